// Instantiations of k_score_tiles: the table-driven cell (FLAVOR 3) with the sparse-output scan (family 8).
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_tabcmp(int qclass)
{
    return qclass == 0 ? k_score_tiles<3, 16, false, false, true> : qclass == 1 ? k_score_tiles<3, 24, false, false, true>
                                                                                : k_score_tiles<3, 32, false, false, true>;
}
