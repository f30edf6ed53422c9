// Instantiations of k_score_tiles: the A/B cells (FLAVOR 0: 2 DPX + 2 IMAD; FLAVOR 2: symmetric potential).
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_f0f2(int family, int qclass)
{
    if (family == 0) return qclass == 0 ? k_score_tiles<0, 16, false> : qclass == 1 ? k_score_tiles<0, 24, false> : k_score_tiles<0, 32, false>;
    return qclass == 0 ? k_score_tiles<2, 16, false> : qclass == 1 ? k_score_tiles<2, 24, false> : k_score_tiles<2, 32, false>;
}
