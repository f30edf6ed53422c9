// Instantiations of k_score_tiles: sparse similarity overrides as corrections of the compare-based cell.
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_ov(int qclass)
{
    return qclass == 0 ? k_score_tiles<1, 16, true> : qclass == 1 ? k_score_tiles<1, 24, true> : k_score_tiles<1, 32, true>;
}
