// Instantiations of k_score_tiles: words of up to 64 symbols (block-wise path for chunks longer than 24), with and
// without the sparse-output scan.
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_wide(bool cmp)
{
    return cmp ? k_score_tiles<1, 24, false, true, true> : k_score_tiles<1, 24, false, true, false>;
}
