// Instantiations of k_score_tiles: the table-driven cell (FLAVOR 3) over words of up to 64 symbols (block-wise path
// for chunks longer than 24), without and with the sparse-output scan (families 9 and 10).
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_tabwide(bool cmp)
{
    return cmp ? k_score_tiles<3, 24, false, true, true> : k_score_tiles<3, 24, false, true, false>;
}
