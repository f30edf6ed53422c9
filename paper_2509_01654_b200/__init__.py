"""B200-native all-pairs Needleman-Wunsch scoring (the hot path of arXiv 2509.01654's
``phonsim``): hand-written sm_100a CUDA behind a C ABI, with a host layer that
keeps the reference's ``compute_all_pairs`` entry point."""
from .host_types import (ComputePlan, ComputeStats, DataError, EncodedWord, PhonsimError,
                         ScoringScheme, DEFAULT_SCHEME)
from .triangle import col_of, edges_before_row, index_of, num_edges, row_of
from .engine import NwapContext, compute_all_pairs, pack_words, preflight_range_check
from .store import EdgeStoreManifest, PipelinedEdgeStoreWriter, load_words, save_words, words_digest

__all__ = [
    "ComputePlan", "ComputeStats", "DataError", "EncodedWord", "PhonsimError", "ScoringScheme",
    "DEFAULT_SCHEME", "NwapContext", "compute_all_pairs", "pack_words", "preflight_range_check",
    "num_edges", "edges_before_row", "row_of", "col_of", "index_of",
    "EdgeStoreManifest", "PipelinedEdgeStoreWriter", "load_words", "save_words", "words_digest",
]
__version__ = "0.1.0"
