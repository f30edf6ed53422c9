// Instantiations of k_score_tiles: the default cell (FLAVOR 1: 2 DPX + IMAD + IADD), uniform schemes.
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_f1(int qclass)
{
    return qclass == 0 ? k_score_tiles<1, 16, false> : qclass == 1 ? k_score_tiles<1, 24, false> : k_score_tiles<1, 32, false>;
}
