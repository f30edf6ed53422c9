/*
 * nwap.h -- C ABI of libnwap.so: all-pairs Needleman-Wunsch scoring of
 * symbol-encoded words on NVIDIA B200 (sm_100a).
 *
 * This is the drop-in boundary for ONE path of the reference package `phonsim`
 * (arXiv 2509.01654): everything `phonsim.engine.compute_all_pairs` does
 * between "words are packed" and "bytes are handed to the sink".  Plain
 * pointers and sizes only; no torch / numpy types.  Each entry point names the
 * reference interface it replaces (paths under pkg/src/phonsim/).
 *
 * Conventions
 *   - every function returns 0 on success or a negative NWAP_E* code; the text
 *     of the last error on the calling thread is nwap_last_error().
 *   - "dev" pointers are device memory on the context's GPU, "host" pointers
 *     are host memory (pinned if you want copies to overlap).
 *   - the library borrows every pointer for the duration of the call only,
 *     except that nwap_create copies the word store into the context.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *     Calls that return host-visible results synchronise that stream.
 *   - a context is bound to one GPU and is not thread-safe; distinct contexts
 *     are independent (one per GPU / per rank).
 *   - linear edge index k <-> (row r, col c), r < c, row-major upper triangle:
 *     k = r*(2n-r-1)/2 + (c-r-1)            (triangle.py:43-46, :86-90)
 *     output byte k-start = (int8) nw_score(word r, word c)   (engine.py:190-191)
 */
#ifndef NWAP_H
#define NWAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NWAP_OK          0
#define NWAP_EINVAL     -1   /* bad argument            -> ValueError  */
#define NWAP_ERANGE     -2   /* int8 overflow preflight -> DataError   */
#define NWAP_ECUDA      -3   /* CUDA runtime failure    -> RuntimeError */
#define NWAP_ENOMEM     -4
#define NWAP_ECAPACITY  -5   /* compaction output buffer too small */

/* kernel variants selectable per call (nwap_score_range `variant`) */
#define NWAP_VARIANT_AUTO    0  /* the packed DPX tile kernel: PACKED3 for a uniform scheme, PACKED_TAB for an override
                                 * scheme; words of 25/33..64 symbols (64: gap -1, engine.py:83-90) run the wide build of
                                 * either.  Only a vocabulary with a word over 64 symbols -- which the preflight admits for
                                 * gap 0 alone -- falls back to SIMPLE. */
#define NWAP_VARIANT_SIMPLE  1  /* one thread per pair, int32 cells, K x K table: any scheme, any q <= 255; the independent
                                 * second implementation the packed kernel is cross-checked against */
#define NWAP_VARIANT_PACKED  2  /* s16x2 DPX tile kernel, 2 DPX + 2 IMAD per packed cell */
#define NWAP_VARIANT_PACKED3 3  /* s16x2 DPX tile kernel, 2 DPX + 1 IMAD + 1 IADD per packed cell; word length <= 64
                                 * (chunks longer than 24 symbols are scored block-wise, 16 columns at a time) */
#define NWAP_VARIANT_PACKED_TAB 5 /* s16x2 DPX tile kernel with a K x K similarity table in shared memory (K <= 256):
                                   * any override table, word length <= 64; one 16-bit load from a row-pair profile (or
                                   * two byte loads from the table) per packed cell instead of compare + multiply */
#define NWAP_VARIANT_PACKED_SYM 4 /* s16x2 DPX tile kernel, symmetric gap potential: 2 DPX + 1 IADD3 per packed cell
                                   * (needs match >= mismatch and no overrides) */

typedef struct nwap_ctx nwap_ctx;

/* Summary statistics of a scored range.  Replaces the (sum, min, max) tuple of
 * engine.py:190-195 and feeds ComputeStats (engine.py:284-290).  `hist[b]`
 * counts scores equal to b-128 (store.py:352-366, raw mode); it is filled only
 * when requested.  An empty range gives sum=0,count=0,min=127,max=-128 -- the
 * accumulator seeds of engine.py:246-247. */
typedef struct nwap_stats {
    int64_t  sum;
    int64_t  count;
    int32_t  min;
    int32_t  max;
    uint64_t hist[256];
} nwap_stats;

const char *nwap_version(void);
const char *nwap_last_error(void);

/* Number of CUDA devices visible; <0 on error. */
int nwap_device_count(void);

/* engine.py:72-96 preflight_range_check.  lengths: host (n,) uint8.
 * Returns q = max word length (>0), NWAP_EINVAL for an empty list, or
 * NWAP_ERANGE with *lo_out / *hi_out = the offending bounds. */
int nwap_preflight(const uint8_t *lengths, int64_t n, int gap, int min_sim, int max_sim,
                   int64_t *lo_out, int64_t *hi_out);

/* engine.py:99-107 _pack_words + engine.py:110-117 _similarity_matrix.
 * ids: host (n, q_stride) uint8 row-major, right padding ignored;
 * lengths: host (n,) uint8, every length in [1, q_stride].
 * Copies the store to `device`, laid out (n, q_pad) with q_pad = 16*ceil(q/16).
 * Runs the preflight; a scheme that could overflow int8 is NWAP_ERANGE. */
int nwap_create(nwap_ctx **ctx_out, int device,
                const uint8_t *ids, int64_t n, int q_stride, const uint8_t *lengths,
                int match, int mismatch, int gap);

/* ScoringScheme.overrides (aligner.py:51-65, engine.py:113-116): install a
 * dense symmetric K x K similarity table (host int8, row-major).  Symbols >= K
 * are rejected.  The packed tile kernel runs the table through its table-driven flavour
 * (NWAP_VARIANT_PACKED_TAB, what NWAP_VARIANT_AUTO picks; K <= 256, words of up to 64 symbols); a table
 * that is the uniform scheme plus at most 2 overrides per symbol (K <= 128, words of up to 32 symbols) can
 * also run as corrections of the compare-based cell (NWAP_VARIANT_PACKED3). */
int nwap_set_similarity(nwap_ctx *ctx, const int8_t *sim, int K);

void nwap_destroy(nwap_ctx *ctx);

/* nwap_destroy returns the context's host-destination pipeline (two device slabs, two streams,
 * four events) and its small device arrays to a per-device cache, so the create -> score ->
 * destroy cycle of the reference-shaped entry point costs no driver allocation after the first
 * call.  nwap_trim() frees everything cached, on every device. */
void nwap_trim(void);

int64_t nwap_num_words(const nwap_ctx *ctx);
int64_t nwap_num_edges(const nwap_ctx *ctx);   /* triangle.py:36-40 */
int     nwap_max_len(const nwap_ctx *ctx);
/* DP cell updates (len_r * len_c summed) inside linear range [start, end). */
int64_t nwap_cells_in_range(const nwap_ctx *ctx, int64_t start, int64_t end);

/* engine.py:176-195 _score_range, the operator seam.
 * Scores edges [start, end) into out_dev[0 .. end-start) (int8, device) and
 * returns the range's statistics in *stats_host (may be NULL: then nothing is
 * synchronised and statistics stay on the device until nwap_read_stats).
 * want_hist != 0 also fills stats->hist. */
int nwap_score_range(nwap_ctx *ctx, int64_t start, int64_t end, int8_t *out_dev,
                     nwap_stats *stats_host, int want_hist, int variant, void *stream);

/* Same seam with a HOST destination: compute in device slabs, copy each slab
 * back while the next one is computed (two streams, two slabs).  out_host
 * should be pinned for the copies to overlap.  This is the call the
 * end-to-end number is measured through. */
int nwap_score_range_host(nwap_ctx *ctx, int64_t start, int64_t end, int8_t *out_host,
                          nwap_stats *stats_host, int want_hist, int variant);

/* The same call split in two, so a caller can consume slab k (sink.write, engine.py:256) while
 * the device scores and copies slab k+1 into another host buffer: _begin enqueues the whole
 * range and returns immediately; _wait blocks until out_host is complete and returns the
 * statistics.  One call in flight per context; out_host must stay valid until _wait. */
int nwap_score_range_host_begin(nwap_ctx *ctx, int64_t start, int64_t end, int8_t *out_host,
                                int want_hist, int variant);
int nwap_score_range_host_wait(nwap_ctx *ctx, nwap_stats *stats_host);

/* Statistics of the most recent asynchronous nwap_score_range on `stream`. */
int nwap_read_stats(nwap_ctx *ctx, nwap_stats *stats_host, void *stream);

/* Statistics (sum/min/max/count/hist) recomputed from a dense payload slice on
 * the device: an independent check of the fused statistics and the on-device
 * form of store.py:342-381 histogram (raw mode). */
int nwap_payload_stats(nwap_ctx *ctx, const int8_t *payload_dev, int64_t count,
                       nwap_stats *stats_host, void *stream);

/* Score-threshold compaction of an already scored slice payload_dev[0..end-start)
 * (keep-mask of graph.py:97-98 with the raw score as the weight):
 * kept edges, in increasing linear index, go to idx_out_dev (int64 absolute
 * index) / score_out_dev (int8); *count_host = number kept (even if > cap, in
 * which case NWAP_ECAPACITY is returned and only the first `cap` are written).
 * degree_dev, if non-NULL, is an (n,) int32 array that gets +1 at both
 * endpoints of every kept edge (graph.py:99-101); it is NOT zeroed here. */
int nwap_compact_range(nwap_ctx *ctx, const int8_t *payload_dev, int64_t start, int64_t end,
                       int threshold, int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap,
                       int64_t *count_host, int32_t *degree_dev, void *stream);

/* The edge writer with score-threshold compaction fused in (BASELINE north_star, kernel K4; keep-mask of
 * graph.py:91-101 applied where the scores are produced): scores [start, end) exactly as nwap_score_range and
 * returns the kept edges -- raw score >= threshold -- in increasing linear index in idx_out_dev (int64) /
 * score_out_dev (int8), *count_host = number kept.  The dense payload is OPTIONAL: with out_dev == NULL no
 * per-edge byte is written to memory at all, so a 600,000-word job (1.8e11 edges) needs no 180 GB buffer and
 * runs on one GPU in one call.  The tile kernel appends kept edges as unordered 64-bit keys; a radix sort
 * restores index order, so the result is identical to nwap_compact_range over the dense payload.
 * degree_dev as for nwap_compact_range (not zeroed here); stats_host (may be NULL) receives the range's
 * sum/min/max/count.  More than `cap` (< 2^31) kept edges: NWAP_ECAPACITY, *count_host is the true count and
 * the output arrays are unspecified.  idx_out_dev doubles as sort scratch.  variant: AUTO, PACKED3 (uniform
 * schemes) or PACKED_TAB (override schemes).  Synchronises `stream`. */
int nwap_score_range_compact(nwap_ctx *ctx, int64_t start, int64_t end, int8_t *out_dev, int threshold,
                             int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap, int64_t *count_host,
                             int32_t *degree_dev, nwap_stats *stats_host, int variant, void *stream);

/* The same with the normalised-weight predicate of graph.py:96-98 (lo <= 100.0*score/max(len_r,len_c) <= hi in
 * IEEE double, as nwap_filter_normalized). */
int nwap_score_range_filter_normalized(nwap_ctx *ctx, int64_t start, int64_t end, int8_t *out_dev, double lo, double hi,
                                       int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap, int64_t *count_host,
                                       int32_t *degree_dev, nwap_stats *stats_host, int variant, void *stream);

/* graph.py:91-101 filter_view keep-mask on the device: keep the edges of an already scored
 * slice whose NORMALISED weight w = 100.0 * score / max(len_r, len_c) satisfies
 * lo <= w <= hi, evaluated in IEEE double exactly as numpy does (graph.py:96-98).
 * Outputs and degree as for nwap_compact_range; lo > hi is NWAP_EINVAL (graph.py:86-87). */
int nwap_filter_normalized(nwap_ctx *ctx, const int8_t *payload_dev, int64_t start, int64_t end,
                           double lo, double hi, int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap,
                           int64_t *count_host, int32_t *degree_dev, void *stream);

/* store.py:342-381 histogram(normalized=True): counts_dev[v + 12800] += 1 for
 * v = floor(100*score / max(len_r, len_c)) (exact integer floor division, store.py:360);
 * counts_dev is a (25501,) uint64 device array, NOT zeroed here.  Asynchronous on `stream`. */
#define NWAP_NHIST_BINS 25501
#define NWAP_NHIST_FIRST (-12800)
int nwap_hist_normalized(nwap_ctx *ctx, const int8_t *payload_dev, int64_t start, int64_t end,
                         uint64_t *counts_dev, void *stream);

/* split [0, num_edges) into `parts` contiguous ranges of equal DP
 * cells.  bounds_out has parts+1 entries, bounds_out[0]=0, bounds_out[parts]=P.
 * Host-side arithmetic only. */
int nwap_equal_work_bounds(const nwap_ctx *ctx, int parts, int64_t *bounds_out);

/* Device-side index recovery, exposed for parity tests of
 * triangle.py:93-112 rows_of_array / cols_of_array: idx_dev (count,) int64 ->
 * rows_dev, cols_dev (count,) int64. */
int nwap_rows_cols(int64_t n, const int64_t *idx_dev, int64_t count,
                   int64_t *rows_dev, int64_t *cols_dev, void *stream);

/* Instruction-issue probes used to state the integer roofline.
 * which: see NWAP_PROBE_*.  Returns warp-instructions per SM per clock in
 * *ipc_out (from in-kernel cycle counters) and wall milliseconds in *ms_out. */
#define NWAP_PROBE_VIADDMNMX_U16X2 0
#define NWAP_PROBE_VIMNMX3_S16X2   1
#define NWAP_PROBE_VIMNMX_S16X2    2
#define NWAP_PROBE_IMAD            3
#define NWAP_PROBE_LOP3            4
#define NWAP_PROBE_IADD3           5
#define NWAP_PROBE_MIX_2ALU_2IMAD  6   /* the packed cell's instruction mix: 2 DPX + 2 IMAD */
#define NWAP_PROBE_MIX_3ALU_1IMAD  7
/* 8..21: single-op and two-pipe mixes used to establish the port model
 * (add.u16x2, min.u16x2, fma.f16x2, max.f16x2, prmt, DPX+IADD, DPX+VIMNMX2, IMAD+IADD,
 *  IMAD+HFMA2, DPX+IMAD, alternative cell formulations, VIADDMNMX+VIMNMX3) -- names in
 * paper_2509_01654_b200/_native.py:PROBES. */
#define NWAP_PROBE_COUNT           30
int nwap_probe(int device, int which, int iters, double *ipc_out, double *ms_out);

/* Kernels launched by this library on the calling process so far. */
int64_t nwap_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* NWAP_H */
