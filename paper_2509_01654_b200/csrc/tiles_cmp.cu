// Instantiations of k_score_tiles: sparse-output mode (threshold compaction fused into the edge writer).
#include "nwap_tile.cuh"
nwap_tile_kernel_t nwap_tiles_cmp(int qclass)
{
    return qclass == 0 ? k_score_tiles<1, 16, false, false, true> : qclass == 1 ? k_score_tiles<1, 24, false, false, true>
                                                                                : k_score_tiles<1, 32, false, false, true>;
}
