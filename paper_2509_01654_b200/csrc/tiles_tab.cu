// Instantiations of k_score_tiles: dense similarity tables (FLAVOR 3, table-driven cell).
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_tab(int qclass)
{
    return qclass == 0 ? k_score_tiles<3, 16, false> : qclass == 1 ? k_score_tiles<3, 24, false> : k_score_tiles<3, 32, false>;
}
