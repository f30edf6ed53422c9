// nwap.cu -- C ABI (include/nwap.h) over the sm_100a kernels in nwap_kernels.cuh.
//
// Host-side responsibilities: own the device copy of the word store, choose the
// kernel variant, enumerate work units, reset/read statistics, slab pipelining
// for host destinations, equal-work shard bounds.  No CPU scoring path exists
// here: every score is produced by a CUDA kernel or the call fails.
#include <algorithm>
#include <memory>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <chrono>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/nwap.h"
#include "nwap_kernels.cuh"

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(NWAP_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

// Every entry point works on its context's GPU and puts the caller's current device back on return: a host
// process that also drives torch (or other contexts) must not find its current device changed behind its back.
struct device_guard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit device_guard(int dev)
    {
        int cur = -1;
        err = cudaGetDevice(&cur);
        if (err == cudaSuccess && cur != dev) {
            err = cudaSetDevice(dev);
            if (err == cudaSuccess) prev = cur;
        }
    }
    ~device_guard() { if (prev >= 0) cudaSetDevice(prev); }
    device_guard(const device_guard &) = delete;
    device_guard &operator=(const device_guard &) = delete;
};
#define ON_DEVICE(dev) device_guard guard_(dev); CK(guard_.err)

static_assert(sizeof(nwap_dev_stats) == sizeof(nwap_stats), "stats layouts must agree");
static_assert(sizeof(nwap_tile_smem_t<1>) <= 227 * 1024 && sizeof(nwap_tile_smem_t<2>) <= 227 * 1024 &&
              sizeof(nwap_tile_smem_t<2, NWAP_MAXLEN_WIDE>) <= 227 * 1024, "tile shared memory too large");
static_assert(2 * sizeof(nwap_tile_smem_t<0, NWAP_MAXLEN_WIDE>) <= 226 * 1024, "the wide build must keep two CTAs per SM");

}  // namespace

nwap_tile_kernel_t nwap_tile_kernel(int family, int qclass)
{
    switch (family) {
    case 0: case 2: return nwap_tiles_f0f2(family, qclass);
    case 3: return nwap_tiles_ov(qclass);
    case 4: return nwap_tiles_tab(qclass);
    case 5: return nwap_tiles_wide(false);
    case 6: return nwap_tiles_cmp(qclass);
    case 7: return nwap_tiles_wide(true);
    case 8: return nwap_tiles_tabcmp(qclass);
    case 9: return nwap_tiles_tabwide(false);
    case 10: return nwap_tiles_tabwide(true);
    default: return nwap_tiles_f1(qclass);
    }
}

typedef nwap_tile_smem_t<2, NWAP_MAXLEN_WIDE> nwap_tile_smem_wide_tab;
static bool nwap_family_is_tab(int family) { return family == 4 || family >= 8; }

size_t nwap_tile_smem_bytes(int family, int K)
{
    switch (family) {
    case 3: return sizeof(nwap_tile_smem_t<1>);
    case 4: case 8: case 9: case 10: {
        // the K x K table is the struct's last member: K = 0 asks for the largest alphabet
        const size_t tab = K > 0 ? (((size_t)K * (size_t)K + 15u) & ~size_t(15)) : (size_t)NWAP_TAB_MAXK * NWAP_TAB_MAXK;
        const size_t base = family >= 9 ? offsetof(nwap_tile_smem_wide_tab, etab) : offsetof(nwap_tile_smem_t<2>, etab);
        return base + std::max<size_t>(16, tab);
    }
    case 5: case 7: return sizeof(nwap_tile_smem_t<0, NWAP_MAXLEN_WIDE>);
    default: return sizeof(nwap_tile_smem_t<0>);
    }
}

struct nwap_ctx {
    int device = 0;
    int sm_count = 0;
    int64_t n = 0;
    int qmax = 0;          // longest word
    double long_share = 0; // share of the vocabulary's symbols that sit in words of more than NWAP_WIDE_FROM symbols
    int qpad = 0;          // stored row width (multiple of 16)
    int match = 0, mismatch = 0, gap = 0;
    int K = 0;             // similarity table size (max symbol + 1 unless overridden)
    bool general = false;  // explicit similarity table installed
    bool sparse_ov = false; // ... and it is uniform + at most NWAP_MAX_OV overrides per symbol (packed kernel can run it)
    nwap_ov_row *d_ov = nullptr;
    bool tab_ok = false;    // ... or any table over K <= 256 symbols: the packed kernel's table-driven flavour runs it
    int tab_max = 0;        // the table's maximum M (the table on the device holds M - sim)
    uint8_t *d_etab = nullptr;
    std::vector<uint8_t> h_lens;        // host copy for shard arithmetic
    std::vector<int64_t> h_lenprefix;   // prefix sums of lengths (n+1)
    std::vector<int64_t> h_rowpref;     // h_rowpref[r] = DP cells of rows < r (n+1)
    uint8_t *d_ids = nullptr;
    uint8_t *d_lens = nullptr;          // padded with zeros to a whole number of strips
    int8_t *d_sim = nullptr;            // K x K
    nwap_dev_stats *d_stats = nullptr;
    unsigned long long *d_counter = nullptr;
    // compaction scratch
    long long *d_block_counts = nullptr;
    int64_t block_counts_cap = 0;
    long long *d_total = nullptr;
    // host-destination pipeline: borrowed from the per-device cache on first use, returned in nwap_destroy
    struct nwap_pipe *pipe = nullptr;
    bool host_pending = false;          // nwap_score_range_host_begin issued, nwap_score_range_host_wait not yet
    int occ_tiles[NWAP_TILE_FAMILIES * 3] = {0};    // resident CTAs/SM per (family, qclass) instantiation (nwap_tile_kernel)
    // sparse-output mode: key scratch (second sort buffer), digit table, kept counter, per-length bounds
    unsigned long long *d_keys = nullptr;
    int64_t keys_cap = 0;
    unsigned int *d_sort_table = nullptr;
    int64_t sort_table_cap = 0;
    unsigned long long *d_kept = nullptr;
    short2 *d_kbounds = nullptr;
    short2 *d_ftab = nullptr;          // normalised filter: 512 per-length score bounds (nwap_keep_params::dtab)
};

// Two device slabs, two streams and four events: everything nwap_score_range_host needs to overlap
// scoring with the device->host copies.
struct nwap_pipe {
    int8_t *d_slab[2] = {nullptr, nullptr};
    int64_t slab_bytes = 0;
    cudaStream_t s_compute = nullptr, s_copy = nullptr;
    cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
};

namespace {

// Per-device facts and scratch that outlive a context.  Creating and destroying a context per
// call (what the reference-shaped entry point does) must not pay cudaGetDeviceProperties, twelve
// occupancy queries, two 256 MB cudaMalloc/cudaFree pairs and stream/event creation every time:
// those were 60 % of the end-to-end step.  nwap_trim() releases the cached scratch.
struct device_cache {
    bool ready = false;
    int sm_count = 0;
    int occ_tiles[NWAP_TILE_FAMILIES * 3] = {0};
    std::vector<nwap_pipe *> free_pipes;
};
std::mutex g_cache_mutex;
device_cache g_cache[64];

void destroy_pipe(nwap_pipe *p)
{
    if (!p) return;
    cudaFree(p->d_slab[0]); cudaFree(p->d_slab[1]);
    for (int i = 0; i < 2; ++i) {
        if (p->ev_done[i]) cudaEventDestroy(p->ev_done[i]);
        if (p->ev_free[i]) cudaEventDestroy(p->ev_free[i]);
    }
    if (p->s_compute) cudaStreamDestroy(p->s_compute);
    if (p->s_copy) cudaStreamDestroy(p->s_copy);
    delete p;
}

// Device facts, kernel attributes and the memory-pool policy: once per device per process.
int ensure_device_cache(int device, device_cache **out)
{
    std::lock_guard<std::mutex> lock(g_cache_mutex);
    device_cache &dc = g_cache[device];
    if (!dc.ready) {
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        dc.sm_count = sms;
        // the small per-context arrays come from the stream-ordered pool; keep freed blocks cached
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        unsigned long long keep = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        for (int f = 0; f < NWAP_TILE_FAMILIES; ++f)
            for (int w = 0; w < 3; ++w) {
                nwap_tile_kernel_t k = nwap_tile_kernel(f, w);
                const size_t smem = nwap_tile_smem_bytes(f);
                // the table flavour's launch adds its row-pair profiles (enqueue_score): allow it the whole SM
                CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, nwap_family_is_tab(f) ? 226 * 1024 : (int)smem));
                int occ = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NWAP_THREADS, smem));
                dc.occ_tiles[f * 3 + w] = occ;
            }
        dc.ready = true;
    }
    *out = &dc;
    return NWAP_OK;
}

// Small per-context device arrays: stream-ordered allocations on the legacy stream (the pool keeps
// freed blocks, so a create/destroy cycle costs no driver allocation).
cudaError_t dev_alloc(void *pp, size_t bytes) { return cudaMallocAsync((void **)pp, bytes, 0); }
void dev_free(void *ptr) { if (ptr) cudaFreeAsync(ptr, 0); }

// Borrow the host-destination pipeline (slabs of at least `slab` bytes) from the device cache.
int acquire_pipe(nwap_ctx *c, int64_t slab)
{
    if (!c->pipe) {
        std::lock_guard<std::mutex> lock(g_cache_mutex);
        std::vector<nwap_pipe *> &fp = g_cache[c->device].free_pipes;
        if (!fp.empty()) { c->pipe = fp.back(); fp.pop_back(); }
    }
    if (!c->pipe) {
        nwap_pipe *p = new nwap_pipe();
        cudaError_t e = cudaStreamCreateWithFlags(&p->s_compute, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_copy, cudaStreamNonBlocking);
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&p->ev_done[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_free[i], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) {          // never cache a half-built pipeline
            destroy_pipe(p);
            return fail(NWAP_ECUDA, "creating the host-destination pipeline failed: %s", cudaGetErrorString(e));
        }
        c->pipe = p;
    }
    nwap_pipe *p = c->pipe;
    if (p->slab_bytes < slab) {
        for (int i = 0; i < 2; ++i) { cudaFree(p->d_slab[i]); p->d_slab[i] = nullptr; }
        p->slab_bytes = 0;
        for (int i = 0; i < 2; ++i) {
            const cudaError_t e = cudaMalloc(&p->d_slab[i], slab);
            if (e != cudaSuccess) {
                for (int k = 0; k < 2; ++k) { cudaFree(p->d_slab[k]); p->d_slab[k] = nullptr; }
                return fail(NWAP_ECUDA, "cudaMalloc of a %lld-byte device slab failed: %s", (long long)slab, cudaGetErrorString(e));
            }
        }
        p->slab_bytes = slab;
    }
    return NWAP_OK;
}

int build_sim_table(nwap_ctx *c, const int8_t *sim_host)
{
    if (c->d_sim) { CK(cudaDeviceSynchronize()); dev_free(c->d_sim); c->d_sim = nullptr; }
    CK(dev_alloc(&c->d_sim, (size_t)c->K * c->K));
    CK(cudaMemcpyAsync(c->d_sim, sim_host, (size_t)c->K * c->K, cudaMemcpyHostToDevice, 0));
    return NWAP_OK;
}

int reset_stats(nwap_ctx *c, cudaStream_t st)
{
    k_init_stats<<<1, 256, 0, st>>>(c->d_stats, c->d_counter);
    g_launches++;
    CK(cudaGetLastError());
    return NWAP_OK;
}

int fetch_stats(nwap_ctx *c, nwap_stats *out, cudaStream_t st)
{
    CK(cudaMemcpyAsync(out, c->d_stats, sizeof(nwap_stats), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return NWAP_OK;
}

// Enqueue the scoring of [start, end) into out_dev on `st`.  Statistics accumulate
// into c->d_stats (caller resets).  No synchronisation.  `sparse` (may be NULL) switches the
// tile kernel's writer to sparse output; out_dev may then be NULL (no dense payload).
int enqueue_score(nwap_ctx *c, int64_t start, int64_t end, int8_t *out_dev, int want_hist,
                  int variant, cudaStream_t st, const nwap_sparse_out *sparse = nullptr)
{
    if (start >= end) return NWAP_OK;
    const bool uniform_ok = !c->general || c->sparse_ov;
    const bool fast_ok = uniform_ok && c->qmax <= NWAP_MAXLEN_FAST;
    const bool wide_ok = !c->general && c->qmax <= NWAP_MAXLEN_WIDE;          // block-wise path: uniform schemes only
    const bool tab_ok = c->general && c->tab_ok && c->qmax <= NWAP_MAXLEN_WIDE;   // words over 32 symbols: the wide build of the table cell
    const bool sym_ok = fast_ok && !c->general && nwap_flavor2_ok(c->match, c->mismatch);
    // PACKED3 (2 DPX + IMAD + IADD) is ~8 % faster than PACKED (2 DPX + 2 IMAD) and ~14 % faster than PACKED_SYM
    // (2 DPX + IADD3: one issue fewer, but IADD3 shares the DPX pipe): profiles/r01f_ab_packed_sym.txt
    // override tables: the table-driven cell (6.1 TCUPS whatever the table holds, two CTAs per SM up to ~100 symbols)
    // is at least as fast as the sparse-correction cell (5.1-6.3 TCUPS, profiles/r02b_overrides.txt) whenever the
    // alphabet fits shared memory, so `auto` takes it first.  A uniform scheme never leaves the packed kernel: the preflight admits at
    // most 64 symbols per word (gap -1, engine.py:83-90), which the wide build covers.
    if (variant == NWAP_VARIANT_AUTO)
        variant = tab_ok ? NWAP_VARIANT_PACKED_TAB : (fast_ok || wide_ok) ? NWAP_VARIANT_PACKED3 : NWAP_VARIANT_SIMPLE;
    if (variant == NWAP_VARIANT_PACKED_TAB && !tab_ok)
        return fail(NWAP_EINVAL, "packed_tab kernel needs a similarity table (overrides) with K <= %d and max word length <= %d", NWAP_TAB_MAXK, NWAP_MAXLEN_WIDE);
    if (variant == NWAP_VARIANT_PACKED_SYM && !sym_ok)
        return fail(NWAP_EINVAL, "packed_sym kernel needs a uniform scheme with match >= mismatch and max word length <= %d (have %d%s)",
                    NWAP_MAXLEN_FAST, c->qmax, c->general ? ", similarity overrides" : "");
    if (variant == NWAP_VARIANT_PACKED && !fast_ok)
        return fail(NWAP_EINVAL, "packed kernel needs a uniform scheme (or at most %d overrides per symbol) and max word length <= %d (have %d%s)",
                    NWAP_MAX_OV, NWAP_MAXLEN_FAST, c->qmax, c->general ? ", dense similarity table" : "");
    if (variant == NWAP_VARIANT_PACKED3 && !fast_ok && !wide_ok)
        return fail(NWAP_EINVAL, "packed kernel needs a uniform scheme and max word length <= %d, or at most %d overrides per symbol and max word length <= %d (have %d%s)",
                    NWAP_MAXLEN_WIDE, NWAP_MAX_OV, NWAP_MAXLEN_FAST, c->qmax, c->general ? ", similarity table" : "");
    if (sparse && !((variant == NWAP_VARIANT_PACKED3 && !c->general) || variant == NWAP_VARIANT_PACKED_TAB))
        return fail(NWAP_EINVAL, "sparse output is built for the default packed kernel (uniform schemes) and the table-driven kernel (override schemes)");

    if (variant == NWAP_VARIANT_SIMPLE) {
        nwap_simple_params p;
        p.ids = c->d_ids; p.lens = c->d_lens; p.n = c->n; p.qpad = c->qpad; p.qmax = c->qmax;
        p.start = start; p.end = end; p.out = out_dev; p.sim = c->d_sim; p.K = c->K; p.gap = c->gap;
        p.stats = c->d_stats; p.want_hist = want_hist;
        const size_t smem = (size_t)((c->K * c->K + 15) & ~15) + (size_t)(c->qmax + 1) * NWAP_SIMPLE_THREADS * sizeof(short);
        CK(cudaFuncSetAttribute(k_score_simple, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int64_t pairs = end - start;
        int64_t blocks = (pairs + NWAP_SIMPLE_THREADS - 1) / NWAP_SIMPLE_THREADS;
        blocks = std::min<int64_t>(blocks, (int64_t)c->sm_count * 16);
        k_score_simple<<<(unsigned)blocks, NWAP_SIMPLE_THREADS, smem, st>>>(p);
        g_launches++;
        CK(cudaGetLastError());
        return NWAP_OK;
    }

    const bool tab = variant == NWAP_VARIANT_PACKED_TAB;
    const bool ov = c->general && !tab;               // here: general and not tab implies sparse_ov
    const int flavor = tab ? 3 : variant == NWAP_VARIANT_PACKED_SYM ? 2 : (ov || variant == NWAP_VARIANT_PACKED3) ? 1 : 0;
    // Uniform schemes take the wide build from 25 symbols on: its 24-wide bodies keep the fast2 family and the few
    // longer chunks go block-wise, which beats the 32-wide instantiation (no fast2, spills) by 29 % on a natural
    // vocabulary with a 25..32-symbol tail (tools/q32_bench.py).  The table-driven cell keeps its 32-wide build (+5 %).
    // The exception: a vocabulary MADE of 25..32-symbol words (every chunk would go block-wise: 10.0 against 14.5 TCUPS
    // at a fixed length of 28).  The two builds cross where ~45 % of the cells sit in long chunks; the share of the
    // symbols that belong to long words estimates that.
    const bool mostly_long = c->qmax <= NWAP_MAXLEN_FAST && c->long_share > 0.40;
    const bool wide = !ov && ((flavor == 1 && c->qmax > NWAP_WIDE_FROM && !mostly_long) || (flavor == 3 && c->qmax > NWAP_MAXLEN_FAST));
    const int qclass = wide ? 1 : c->qmax <= 16 ? 0 : c->qmax <= 24 ? 1 : 2;
    const int family = tab ? (wide ? (sparse ? 10 : 9) : sparse ? 8 : 4)
                           : wide ? (sparse ? 7 : 5) : sparse ? 6 : ov ? 3 : flavor;
    nwap_tile_params p;
    p.ids = c->d_ids; p.lens = c->d_lens; p.n = c->n; p.qpad = c->qpad;
    p.start = start; p.end = end;
    p.r_first = nwap_row_of(start, c->n);
    p.c_start = nwap_col_of(start, c->n, p.r_first);
    p.r_last = nwap_row_of(end - 1, c->n);
    p.c_end = nwap_col_of(end - 1, c->n, p.r_last);
    p.out = out_dev;
    p.sc = tab ? nwap_make_consts(c->tab_max, c->tab_max, c->gap, 3) : nwap_make_consts(c->match, c->mismatch, c->gap, flavor);
    if (tab) p.sc.symmul = (uint32_t)c->K;           // staged row symbol = row offset a*K in the table
    p.stats = c->d_stats; p.want_hist = want_hist;
    p.unit_counter = c->d_counter;
    p.ov_table = ov ? c->d_ov : nullptr; p.ov_K = (ov || tab) ? c->K : 0;
    p.etab = tab ? c->d_etab : nullptr;
    if (sparse) p.sparse = *sparse;
    else memset(&p.sparse, 0, sizeof p.sparse);

    int occ = std::max(1, c->occ_tiles[family * 3 + qclass]);
    p.tab2_lmax = 0;
    size_t smem_bytes = nwap_tile_smem_bytes(family, tab ? c->K : 0);
    if (tab) {
        // second shape of the table cell (one load per packed cell): row-pair profiles behind the table, when they fit
        static const bool no_tab2 = getenv("NWAP_NO_TAB2") && atoi(getenv("NWAP_NO_TAB2")) != 0;
        const size_t prof = nwap_tab2_prof_bytes(c->qmax, c->K) + sizeof(nwap_pair_meta) * NWAP_TAB2_PAIRS;
        if (!no_tab2 && smem_bytes + prof <= (size_t)226 * 1024) { smem_bytes += prof; p.tab2_lmax = c->qmax; }
    }
    if (tab) {          // the table-driven flavour's footprint depends on the alphabet: two CTAs per SM up to ~100 symbols
        int o = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, nwap_tile_kernel(family, qclass), NWAP_THREADS, smem_bytes));
        occ = std::max(1, o);
    }
    const int64_t slots = (int64_t)c->sm_count * occ;
    // bands per group: as large as possible (amortises the per-unit sort) while
    // leaving >= 24 units per resident CTA for dynamic balance.
    const int cw = tab ? NWAP_TAB_CW : NWAP_C;              // strip width of the build (nwap_tile_smem_t<..>::C)
    const int bands_per_strip = cw / NWAP_R;
    int gb = 16;
    nwap_unit_space us;
    int64_t ubeg = 0, ucount = 0;
    for (;; gb >>= 1) {
        us.n = c->n; us.S = (c->n + cw - 1) / cw; us.gb = gb; us.gpk = bands_per_strip / gb;
        const int64_t rows_per_group = (int64_t)gb * NWAP_R;
        const int64_t g0 = p.r_first / rows_per_group, g1 = p.r_last / rows_per_group;
        ubeg = nwap_units_before_group(us, g0);
        ucount = nwap_units_before_group(us, g1 + 1) - ubeg;
        if (gb == 1 || ucount >= slots * NWAP_UNITS_PER_SLOT) break;
    }
    p.us = us; p.unit_begin = ubeg; p.unit_count = ucount;
    const int64_t grid = std::min<int64_t>(slots, ucount);
    CK(cudaMemsetAsync(c->d_counter, 0, sizeof(unsigned long long), st));
    nwap_tile_kernel(family, qclass)<<<(unsigned)grid, NWAP_THREADS, smem_bytes, st>>>(p);
    g_launches++;
    CK(cudaGetLastError());
    if (want_hist && out_dev) {
        // the histogram comes from a streaming pass over the bytes just written (still L2-warm for slabs): the
        // scoring kernel keeps its fast emit, and the pass runs at 5.5 TB/s (profiles/r01_consumers_ncu.txt)
        const int64_t count = end - start;
        const int64_t blocks = std::min<int64_t>((count / 16 + 255) / 256 + 1, (int64_t)c->sm_count * 8);
        k_payload_stats<<<(unsigned)blocks, 256, 0, st>>>(out_dev, count, c->d_stats, 1);
        g_launches++;
        CK(cudaGetLastError());
    }
    return NWAP_OK;
}

}  // namespace

extern "C" {

const char *nwap_version(void) { return "nwap 0.1 (sm_100a)"; }
const char *nwap_last_error(void) { return g_err.c_str(); }
int64_t nwap_launch_count(void) { return g_launches.load(); }

int nwap_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return fail(NWAP_ECUDA, "cudaGetDeviceCount failed"); }
    return n;
}

int nwap_preflight(const uint8_t *lengths, int64_t n, int gap, int min_sim, int max_sim,
                   int64_t *lo_out, int64_t *hi_out)
{
    if (n <= 0 || !lengths) return fail(NWAP_EINVAL, "word list is empty");
    int64_t q = 0;
    for (int64_t i = 0; i < n; ++i) q = std::max<int64_t>(q, lengths[i]);
    const int64_t lo = std::min<int64_t>({0, 2 * q * gap, q * min_sim});
    const int64_t hi = std::max<int64_t>({0, 2 * q * gap, q * max_sim});
    if (lo_out) *lo_out = lo;
    if (hi_out) *hi_out = hi;
    if (lo < -128 || hi > 127)
        return fail(NWAP_ERANGE, "scores would overflow 8-bit storage for max word length %lld: bounds [%lld, %lld]",
                    (long long)q, (long long)lo, (long long)hi);
    return (int)q;
}

namespace {
struct phase_timer {
    bool on; std::chrono::steady_clock::time_point t0;
    phase_timer() : on(getenv("NWAP_TIMING") != nullptr), t0(std::chrono::steady_clock::now()) {}
    void mark(const char *what) {
        if (!on) return;
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[nwap timing] %-22s %8.1f us\n", what, std::chrono::duration<double, std::micro>(t1 - t0).count());
        t0 = t1;
    }
};
}

int nwap_create(nwap_ctx **ctx_out, int device, const uint8_t *ids, int64_t n, int q_stride,
                const uint8_t *lengths, int match, int mismatch, int gap)
{
    phase_timer pt;
    if (!ctx_out || !ids || !lengths) return fail(NWAP_EINVAL, "null argument");
    if (n < 2) return fail(NWAP_EINVAL, "need at least two words");
    if (device < 0 || device >= 64) return fail(NWAP_EINVAL, "device %d out of range", device);
    if (q_stride < 1 || q_stride > 255) return fail(NWAP_EINVAL, "q_stride %d out of range [1, 255]", q_stride);
    int q = nwap_preflight(lengths, n, gap, std::min(match, mismatch), std::max(match, mismatch), nullptr, nullptr);
    if (q < 0) return q;
    if (q > q_stride) return fail(NWAP_EINVAL, "a word length (%d) exceeds q_stride (%d)", q, q_stride);
    // one pass over the words: reject empty ones, repack the rows to qpad bytes (zero padded) and find the largest
    // symbol.  16 bytes at a time with a per-length mask where the source row allows it (this pass and the repack
    // were 3.3 of the 3.8 ms a context costs at 100,000 words, all of it inside the end-to-end step).
    const int qpad_ = ((q + 15) / 16) * 16;
    std::unique_ptr<uint8_t[]> packed(new uint8_t[(size_t)n * qpad_]);
    int maxsym = 0;
    {
        const int64_t total = n * (int64_t)q_stride;
        int64_t i = 0;
#if defined(__SSE2__)
        alignas(16) uint8_t mask16[17][16];
        for (int l = 0; l <= 16; ++l) for (int b = 0; b < 16; ++b) mask16[l][b] = b < l ? 0xff : 0x00;
        __m128i mx = _mm_setzero_si128();
        for (; i < n && i * (int64_t)q_stride + qpad_ <= total; ++i) {
            const int len = lengths[i];
            if (len < 1) return fail(NWAP_EINVAL, "word %lld is empty (length 0)", (long long)i);
            const uint8_t *src = ids + i * q_stride;
            uint8_t *dst = packed.get() + (size_t)i * qpad_;
            for (int h = 0; h < qpad_; h += 16) {
                const int lh = std::min(16, std::max(0, len - h));
                const __m128i v = _mm_and_si128(_mm_loadu_si128(reinterpret_cast<const __m128i *>(src + h)),
                                                _mm_load_si128(reinterpret_cast<const __m128i *>(mask16[lh])));
                _mm_storeu_si128(reinterpret_cast<__m128i *>(dst + h), v);
                mx = _mm_max_epu8(mx, v);
            }
        }
        alignas(16) uint8_t mxb[16];
        _mm_store_si128(reinterpret_cast<__m128i *>(mxb), mx);
        for (int b = 0; b < 16; ++b) maxsym = std::max<int>(maxsym, mxb[b]);
#endif
        for (; i < n; ++i) {                                     // the last rows (and hosts without SSE2): bytewise
            const int len = lengths[i];
            if (len < 1) return fail(NWAP_EINVAL, "word %lld is empty (length 0)", (long long)i);
            uint8_t *dst = packed.get() + (size_t)i * qpad_;
            memset(dst, 0, qpad_);
            for (int j = 0; j < len; ++j) { dst[j] = ids[i * q_stride + j]; maxsym = std::max<int>(maxsym, dst[j]); }
        }
    }
    pt.mark("validate");
    ON_DEVICE(device);
    device_cache *dc = nullptr;
    {
        const int rc0 = ensure_device_cache(device, &dc);
        if (rc0) return rc0;
    }
    pt.mark("device cache");
    nwap_ctx *c = new nwap_ctx();
    c->sm_count = dc->sm_count;
    memcpy(c->occ_tiles, dc->occ_tiles, sizeof dc->occ_tiles);
    c->device = device; c->n = n; c->qmax = q; c->qpad = ((q + 15) / 16) * 16;
    c->match = match; c->mismatch = mismatch; c->gap = gap; c->K = maxsym + 1;
    c->h_lens.assign(lengths, lengths + n);
    c->h_lenprefix.resize(n + 1);
    c->h_lenprefix[0] = 0;
    int64_t long_syms = 0;                                      // symbols of the words the 24-wide bodies cannot hold
    for (int64_t i = 0; i < n; ++i) {
        c->h_lenprefix[i + 1] = c->h_lenprefix[i] + lengths[i];
        if (lengths[i] > NWAP_WIDE_FROM) long_syms += lengths[i];
    }
    c->long_share = (double)long_syms / (double)std::max<int64_t>(1, c->h_lenprefix[n]);
    c->h_rowpref.assign(n + 1, 0);
    for (int64_t r = 0; r < n; ++r)
        c->h_rowpref[r + 1] = c->h_rowpref[r] + (int64_t)lengths[r] * (c->h_lenprefix[n] - c->h_lenprefix[r + 1]);

    pt.mark("prefix sums");
    // (rows were repacked to qpad above) one H2D copy
    const size_t packed_bytes = (size_t)n * c->qpad;
    pt.mark("repack");
    const int64_t lens_pad = ((n + NWAP_C - 1) / NWAP_C) * NWAP_C + NWAP_C;
    int rc = NWAP_OK;
    auto guard = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess && rc == NWAP_OK) rc = fail(NWAP_ECUDA, "%s failed: %s", what, cudaGetErrorString(e));
    };
    guard(dev_alloc(&c->d_ids, packed_bytes), "alloc(ids)");
    guard(dev_alloc(&c->d_lens, lens_pad), "alloc(lens)");
    guard(dev_alloc(&c->d_stats, sizeof(nwap_dev_stats)), "alloc(stats)");
    guard(dev_alloc(&c->d_counter, sizeof(unsigned long long)), "alloc(counter)");
    guard(dev_alloc(&c->d_total, sizeof(long long)), "alloc(total)");
    pt.mark("allocs");
    if (rc == NWAP_OK) {
        guard(cudaMemcpyAsync(c->d_ids, packed.get(), packed_bytes, cudaMemcpyHostToDevice, 0), "H2D ids");
        guard(cudaMemsetAsync(c->d_lens, 0, lens_pad, 0), "memset lens");
        guard(cudaMemcpyAsync(c->d_lens, lengths, n, cudaMemcpyHostToDevice, 0), "H2D lens");
    }
    pt.mark("H2D enqueue");
    if (rc == NWAP_OK) {
        // uniform-scheme similarity table (engine.py:110-112) for the generic kernel
        std::vector<int8_t> sim((size_t)c->K * c->K, (int8_t)mismatch);
        for (int k = 0; k < c->K; ++k) sim[(size_t)k * c->K + k] = (int8_t)match;
        rc = build_sim_table(c, sim.data());
    }
    pt.mark("sim table");
    // the store must be complete before kernels on other (non-blocking) streams read it
    if (rc == NWAP_OK) guard(cudaStreamSynchronize(0), "H2D word store");
    pt.mark("sync");
    if (rc != NWAP_OK) { nwap_destroy(c); return rc; }
    *ctx_out = c;
    return NWAP_OK;
}

int nwap_set_similarity(nwap_ctx *c, const int8_t *sim, int K)
{
    if (!c || !sim) return fail(NWAP_EINVAL, "null argument");
    if (K < c->K) return fail(NWAP_EINVAL, "similarity table K=%d smaller than max symbol + 1 = %d", K, c->K);
    if (K > 256) return fail(NWAP_EINVAL, "similarity table K=%d exceeds 256", K);
    int mn = 127, mx = -128;
    for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) {
            if (sim[a * K + b] != sim[b * K + a]) return fail(NWAP_EINVAL, "similarity table is not symmetric at (%d, %d)", a, b);
            mn = std::min<int>(mn, sim[a * K + b]);
            mx = std::max<int>(mx, sim[a * K + b]);
        }
    int q = nwap_preflight(c->h_lens.data(), c->n, c->gap, mn, mx, nullptr, nullptr);
    if (q < 0) return q;
    ON_DEVICE(c->device);
    c->K = K;
    c->general = true;
    // uniform + sparse corrections?  then the packed kernel can run it
    std::vector<nwap_ov_row> tab((size_t)K);
    c->sparse_ov = K <= NWAP_OV_MAXK && nwap_build_ov_table(sim, K, c->match, c->mismatch, tab.data());
    if (c->d_ov) { CK(cudaDeviceSynchronize()); dev_free(c->d_ov); c->d_ov = nullptr; }
    if (c->sparse_ov) {
        CK(dev_alloc(&c->d_ov, sizeof(nwap_ov_row) * (size_t)K));
        CK(cudaMemcpyAsync(c->d_ov, tab.data(), sizeof(nwap_ov_row) * (size_t)K, cudaMemcpyHostToDevice, 0));
    }
    // dense but small alphabet: E = M - sim for the packed kernel's table-driven flavour
    if (c->d_etab) { CK(cudaDeviceSynchronize()); dev_free(c->d_etab); c->d_etab = nullptr; }
    c->tab_ok = K <= NWAP_TAB_MAXK;       // (a sparse table can run either way; `auto` prefers the sparse-override cell)
    std::vector<uint8_t> etab;
    if (c->tab_ok) {
        c->tab_max = mx;
        etab.resize((size_t)K * K);
        for (int i = 0; i < K * K; ++i) etab[i] = (uint8_t)(mx - (int)sim[i]);
        CK(dev_alloc(&c->d_etab, etab.size()));
        CK(cudaMemcpyAsync(c->d_etab, etab.data(), etab.size(), cudaMemcpyHostToDevice, 0));
    }
    const int rc = build_sim_table(c, sim);
    CK(cudaStreamSynchronize(0));        // tab / etab / sim are host temporaries; other streams read the tables
    return rc;
}

void nwap_destroy(nwap_ctx *c)
{
    if (!c) return;
    device_guard guard_(c->device);
    cudaDeviceSynchronize();             // nothing may still be reading the store or writing the slabs
    dev_free(c->d_ids); dev_free(c->d_lens); dev_free(c->d_sim); dev_free(c->d_stats); dev_free(c->d_ov); dev_free(c->d_etab);
    dev_free(c->d_counter); dev_free(c->d_block_counts); dev_free(c->d_total);
    dev_free(c->d_kept); dev_free(c->d_kbounds); dev_free(c->d_ftab);
    cudaFree(c->d_keys); cudaFree(c->d_sort_table);
    if (c->pipe) {                       // back to the device cache for the next context
        std::lock_guard<std::mutex> lock(g_cache_mutex);
        g_cache[c->device].free_pipes.push_back(c->pipe);
    }
    delete c;
}

void nwap_trim(void)
{
    std::lock_guard<std::mutex> lock(g_cache_mutex);
    int cur = 0;
    cudaGetDevice(&cur);
    for (int d = 0; d < 64; ++d) {
        if (g_cache[d].free_pipes.empty()) continue;
        cudaSetDevice(d);
        for (nwap_pipe *p : g_cache[d].free_pipes) destroy_pipe(p);
        g_cache[d].free_pipes.clear();
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    }
    cudaSetDevice(cur);
}

int64_t nwap_num_words(const nwap_ctx *c) { return c ? c->n : 0; }
int64_t nwap_num_edges(const nwap_ctx *c) { return c ? c->n * (c->n - 1) / 2 : 0; }
int nwap_max_len(const nwap_ctx *c) { return c ? c->qmax : 0; }

// cells in rows [0, r) plus the first (c - r - 1) pairs of row r
static int64_t cells_before(const nwap_ctx *c, int64_t idx)
{
    const int64_t n = c->n, P = n * (n - 1) / 2;
    if (idx <= 0) return 0;
    if (idx >= P) return c->h_rowpref[n - 1];
    const std::vector<int64_t> &pre = c->h_lenprefix;
    const int64_t r = nwap_row_of(idx, n);
    const int64_t col = nwap_col_of(idx, n, r);
    return c->h_rowpref[r] + (int64_t)c->h_lens[r] * (pre[col] - pre[r + 1]);
}

int64_t nwap_cells_in_range(const nwap_ctx *c, int64_t start, int64_t end)
{
    if (!c || start >= end) return 0;
    return cells_before(c, end) - cells_before(c, start);
}

int nwap_score_range(nwap_ctx *c, int64_t start, int64_t end, int8_t *out_dev, nwap_stats *stats_host,
                     int want_hist, int variant, void *stream)
{
    if (!c) return fail(NWAP_EINVAL, "null context");
    const int64_t P = nwap_num_edges(c);
    if (start < 0 || end > P || start > end) return fail(NWAP_EINVAL, "range [%lld, %lld) outside [0, %lld)", (long long)start, (long long)end, (long long)P);
    if (start < end && !out_dev) return fail(NWAP_EINVAL, "null output buffer");
    ON_DEVICE(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    int rc = reset_stats(c, st);
    if (rc) return rc;
    rc = enqueue_score(c, start, end, out_dev, want_hist, variant, st);
    if (rc) return rc;
    if (stats_host) return fetch_stats(c, stats_host, st);
    return NWAP_OK;
}

int nwap_read_stats(nwap_ctx *c, nwap_stats *stats_host, void *stream)
{
    if (!c || !stats_host) return fail(NWAP_EINVAL, "null argument");
    ON_DEVICE(c->device);
    return fetch_stats(c, stats_host, (cudaStream_t)stream);
}

int nwap_score_range_host_begin(nwap_ctx *c, int64_t start, int64_t end, int8_t *out_host, int want_hist, int variant)
{
    if (!c) return fail(NWAP_EINVAL, "null context");
    if (c->host_pending) return fail(NWAP_EINVAL, "a host-destination call is already in flight on this context");
    const int64_t P = nwap_num_edges(c);
    if (start < 0 || end > P || start > end) return fail(NWAP_EINVAL, "range [%lld, %lld) outside [0, %lld)", (long long)start, (long long)end, (long long)P);
    if (start < end && !out_host) return fail(NWAP_EINVAL, "null output buffer");
    ON_DEVICE(c->device);
    const int64_t total = end - start;
    // slab: large enough to amortise launches, small enough that the first copy starts early
    int64_t slab = std::max<int64_t>(int64_t(8) << 20, std::min<int64_t>(int64_t(256) << 20, (total + 7) / 8));
    slab = (slab + 255) & ~int64_t(255);
    int rc = acquire_pipe(c, slab);
    if (rc) return rc;
    nwap_pipe *p = c->pipe;
    rc = reset_stats(c, p->s_compute);
    if (rc) return rc;
    // the first two slabs are short (16 MB, 64 MB) so the first device->host copy starts after ~0.1 ms of
    // scoring instead of ~1.7 ms; from then on the copy engine is the bottleneck and never idles
    int k = 0;
    for (int64_t pos = start; pos < end; ++k) {
        const int b = k & 1;
        const int64_t this_slab = k == 0 ? std::min<int64_t>(slab, int64_t(16) << 20)
                                : k == 1 ? std::min<int64_t>(slab, int64_t(64) << 20) : slab;
        const int64_t e = std::min(end, pos + this_slab);
        if (k >= 2) CK(cudaStreamWaitEvent(p->s_compute, p->ev_free[b], 0));
        rc = enqueue_score(c, pos, e, p->d_slab[b], want_hist, variant, p->s_compute);
        if (rc) { cudaStreamSynchronize(p->s_compute); cudaStreamSynchronize(p->s_copy); return rc; }
        CK(cudaEventRecord(p->ev_done[b], p->s_compute));
        CK(cudaStreamWaitEvent(p->s_copy, p->ev_done[b], 0));
        CK(cudaMemcpyAsync(out_host + (pos - start), p->d_slab[b], (size_t)(e - pos), cudaMemcpyDeviceToHost, p->s_copy));
        CK(cudaEventRecord(p->ev_free[b], p->s_copy));
        pos = e;
    }
    c->host_pending = true;
    return NWAP_OK;
}

int nwap_score_range_host_wait(nwap_ctx *c, nwap_stats *stats_host)
{
    if (!c) return fail(NWAP_EINVAL, "null context");
    if (!c->host_pending) return fail(NWAP_EINVAL, "no host-destination call in flight on this context");
    c->host_pending = false;
    ON_DEVICE(c->device);
    nwap_pipe *p = c->pipe;
    CK(cudaStreamSynchronize(p->s_copy));
    if (stats_host) return fetch_stats(c, stats_host, p->s_compute);
    CK(cudaStreamSynchronize(p->s_compute));
    return NWAP_OK;
}

int nwap_score_range_host(nwap_ctx *c, int64_t start, int64_t end, int8_t *out_host, nwap_stats *stats_host,
                          int want_hist, int variant)
{
    const int rc = nwap_score_range_host_begin(c, start, end, out_host, want_hist, variant);
    if (rc) return rc;
    return nwap_score_range_host_wait(c, stats_host);
}

int nwap_payload_stats(nwap_ctx *c, const int8_t *payload_dev, int64_t count, nwap_stats *stats_host, void *stream)
{
    if (!c || !stats_host) return fail(NWAP_EINVAL, "null argument");
    if (count < 0 || (count > 0 && !payload_dev)) return fail(NWAP_EINVAL, "bad payload");
    ON_DEVICE(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    int rc = reset_stats(c, st);
    if (rc) return rc;
    if (count > 0) {
        int64_t blocks = std::min<int64_t>((count / 16 + 255) / 256 + 1, (int64_t)c->sm_count * 8);
        k_payload_stats<<<(unsigned)blocks, 256, 0, st>>>(payload_dev, count, c->d_stats, 0);
        g_launches++;
        CK(cudaGetLastError());
    }
    return fetch_stats(c, stats_host, st);
}

static int compact_common(nwap_ctx *c, const int8_t *payload_dev, int64_t start, int64_t end, int mode,
                          const nwap_keep_params &kp_in, int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap,
                          int64_t *count_host, int32_t *degree_dev, cudaStream_t st)
{
    if (!c || !count_host) return fail(NWAP_EINVAL, "null argument");
    const int64_t P = nwap_num_edges(c);
    if (start < 0 || end > P || start > end) return fail(NWAP_EINVAL, "range [%lld, %lld) outside [0, %lld)", (long long)start, (long long)end, (long long)P);
    if (cap < 0 || (cap > 0 && (!idx_out_dev || !score_out_dev))) return fail(NWAP_EINVAL, "bad output buffers");
    *count_host = 0;
    const int64_t count = end - start;
    if (count == 0) return NWAP_OK;
    if (!payload_dev) return fail(NWAP_EINVAL, "null payload");
    ON_DEVICE(c->device);
    nwap_keep_params kp = kp_in;
    kp.dtab = nullptr;
    if (mode == 1) {
        if (!c->d_ftab) CK(dev_alloc(&c->d_ftab, sizeof(short2) * 512));
        short2 hb[512];
        for (int m = 0; m < 256; ++m) {
            hb[m] = make_short2(kp.smin[m], kp.smax[m]);
            hb[256 + m] = make_short2(kp.rmin[m], kp.rmax[m]);
        }
        CK(cudaMemcpyAsync(c->d_ftab, hb, sizeof hb, cudaMemcpyHostToDevice, st));   // pageable source: staged before return
        kp.dtab = c->d_ftab;
    }
    // blocks tile the 16-byte aligned window that contains the slice (k_compact_*: nwap_cmp_first)
    const int64_t lead = (int64_t)(reinterpret_cast<uintptr_t>(payload_dev) & 15u);
    const int64_t nblocks = (lead + count + NWAP_CMP_BLOCK - 1) / NWAP_CMP_BLOCK;
    if (nblocks > 0x7fffffffLL) return fail(NWAP_EINVAL, "range too large for one compaction call; split it");
    if (c->block_counts_cap < nblocks) {
        CK(cudaDeviceSynchronize());     // an earlier compaction on another stream may still use the old scratch
        dev_free(c->d_block_counts); c->d_block_counts = nullptr;
        // block counts, then one total per scan group behind them
        CK(dev_alloc(&c->d_block_counts, sizeof(long long) * (size_t)(nblocks + (nblocks + NWAP_SCAN_GROUP - 1) / NWAP_SCAN_GROUP)));
        CK(cudaStreamSynchronize(0));
        c->block_counts_cap = nblocks;
    }
    const int64_t ngroups = (nblocks + NWAP_SCAN_GROUP - 1) / NWAP_SCAN_GROUP;
    unsigned long long *group_totals = reinterpret_cast<unsigned long long *>(c->d_block_counts + c->block_counts_cap);
    CK(cudaMemsetAsync(group_totals, 0, sizeof(unsigned long long) * (size_t)ngroups, st));
    if (mode == 0) k_compact_count<0><<<(unsigned)nblocks, NWAP_CMP_THREADS, 0, st>>>(payload_dev, count, kp, c->d_block_counts, group_totals);
    else k_compact_count<1><<<(unsigned)nblocks, NWAP_CMP_THREADS, 0, st>>>(payload_dev, count, kp, c->d_block_counts, group_totals);
    k_compact_scan<<<(unsigned)ngroups, 1024, 0, st>>>(c->d_block_counts, nblocks, group_totals, ngroups, c->d_total);
    if (mode == 0) k_compact_write<0><<<(unsigned)nblocks, NWAP_CMP_THREADS, 0, st>>>(payload_dev, count, kp, c->d_block_counts, c->d_total, nblocks, idx_out_dev, score_out_dev, cap, degree_dev);
    else k_compact_write<1><<<(unsigned)nblocks, NWAP_CMP_THREADS, 0, st>>>(payload_dev, count, kp, c->d_block_counts, c->d_total, nblocks, idx_out_dev, score_out_dev, cap, degree_dev);
    g_launches += 3;
    CK(cudaGetLastError());
    long long total = 0;
    CK(cudaMemcpyAsync(&total, c->d_total, sizeof total, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *count_host = total;
    if (total > cap) return fail(NWAP_ECAPACITY, "compaction kept %lld edges but capacity is %lld", total, (long long)cap);
    return NWAP_OK;
}

int nwap_compact_range(nwap_ctx *c, const int8_t *payload_dev, int64_t start, int64_t end, int threshold,
                       int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap, int64_t *count_host,
                       int32_t *degree_dev, void *stream)
{
    if (!c) return fail(NWAP_EINVAL, "null context");
    nwap_keep_params kp;
    memset(&kp, 0, sizeof kp); kp.threshold = threshold; kp.lens = c->d_lens; kp.n = c->n; kp.start = start;
    return compact_common(c, payload_dev, start, end, 0, kp, idx_out_dev, score_out_dev, cap, count_host, degree_dev,
                          (cudaStream_t)stream);
}

// Sparse-output scoring (the edge writer with threshold compaction fused in): score [start, end), keep what the
// predicate keeps, restore index order, unpack.  mode 1: raw threshold, mode 2: normalised-weight bounds.
static int score_sparse_common(nwap_ctx *c, int64_t start, int64_t end, int8_t *out_dev, int mode, int threshold,
                               double lo, double hi, int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap,
                               int64_t *count_host, int32_t *degree_dev, nwap_stats *stats_host, int variant,
                               cudaStream_t st)
{
    if (!c || !count_host) return fail(NWAP_EINVAL, "null argument");
    const int64_t P = nwap_num_edges(c);
    if (start < 0 || end > P || start > end) return fail(NWAP_EINVAL, "range [%lld, %lld) outside [0, %lld)", (long long)start, (long long)end, (long long)P);
    if (cap < 0 || cap > 0x7fffffffLL || (cap > 0 && (!idx_out_dev || !score_out_dev))) return fail(NWAP_EINVAL, "bad output buffers (capacity must be in [0, 2^31))");
    if (P >= (int64_t(1) << 55)) return fail(NWAP_EINVAL, "too many edges for the 56-bit index keys of the sparse output");
    *count_host = 0;
    ON_DEVICE(c->device);
    if (!c->d_kept) {
        CK(dev_alloc(&c->d_kept, sizeof(unsigned long long)));
        CK(dev_alloc(&c->d_kbounds, sizeof(short2) * 256));
    }
    if (c->keys_cap < cap) {
        CK(cudaDeviceSynchronize());
        cudaFree(c->d_keys); c->d_keys = nullptr; c->keys_cap = 0;
        if (cudaMalloc(&c->d_keys, sizeof(unsigned long long) * (size_t)cap) != cudaSuccess) {
            cudaGetLastError();
            return fail(NWAP_ENOMEM, "cudaMalloc of the %lld-entry key scratch failed", (long long)cap);
        }
        c->keys_cap = cap;
    }
    nwap_sparse_out so;
    memset(&so, 0, sizeof so);
    so.mode = mode; so.threshold = threshold; so.keys = reinterpret_cast<unsigned long long *>(idx_out_dev);
    so.cap = cap; so.count = c->d_kept; so.degree = degree_dev; so.bounds = c->d_kbounds;
    if (mode == 2) {
        nwap_keep_params kp;
        nwap_fill_norm_bounds(kp, lo, hi);
        short2 hb[256];
        for (int m = 0; m < 256; ++m) hb[m] = make_short2(kp.smin[m], kp.smax[m]);
        so.gmin = kp.gmin; so.gmax = kp.gmax;
        CK(cudaMemcpyAsync(c->d_kbounds, hb, sizeof hb, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));          // hb is a stack temporary
    }
    int rc = reset_stats(c, st);
    if (rc) return rc;
    CK(cudaMemsetAsync(c->d_kept, 0, sizeof(unsigned long long), st));
    rc = enqueue_score(c, start, end, out_dev, 0, variant, st, &so);
    if (rc) return rc;
    unsigned long long kept = 0;
    CK(cudaMemcpyAsync(&kept, c->d_kept, sizeof kept, cudaMemcpyDeviceToHost, st));
    if (stats_host) { rc = fetch_stats(c, stats_host, st); if (rc) return rc; }
    else CK(cudaStreamSynchronize(st));
    *count_host = (int64_t)kept;
    if ((int64_t)kept > cap) return fail(NWAP_ECAPACITY, "sparse output kept %lld edges but capacity is %lld", (long long)kept, (long long)cap);
    if (kept == 0) return NWAP_OK;
    // restore index order: LSD radix sort of the index bits (the low 8 bits of a key are the score)
    const long long n = (long long)kept;
    long long tile = NWAP_SORT_TILE;
    if ((n + tile - 1) / tile > 65536) tile = (((n + 65535) / 65536) + 31) / 32 * 32;
    const long long ntiles = (n + tile - 1) / tile;
    if (c->sort_table_cap < 256 * ntiles) {
        CK(cudaDeviceSynchronize());
        cudaFree(c->d_sort_table); c->d_sort_table = nullptr; c->sort_table_cap = 0;
        if (cudaMalloc(&c->d_sort_table, sizeof(unsigned int) * (size_t)(256 * ntiles)) != cudaSuccess) {
            cudaGetLastError();
            return fail(NWAP_ENOMEM, "cudaMalloc of the sort table failed");
        }
        c->sort_table_cap = 256 * ntiles;
    }
    int bits = 1;
    while (bits < 55 && (int64_t(1) << bits) < P) ++bits;
    unsigned long long *src = so.keys, *dst = c->d_keys;
    const unsigned sblocks = (unsigned)((ntiles + NWAP_SORT_WARPS - 1) / NWAP_SORT_WARPS);
    for (int shift = 8; shift < 8 + bits; shift += 8) {
        k_sort_hist<<<sblocks, NWAP_SORT_WARPS * 32, 0, st>>>(src, n, shift, c->d_sort_table, ntiles, tile);
        k_sort_scan<<<1, 1024, 0, st>>>(c->d_sort_table, 256 * ntiles);
        k_sort_scatter<<<sblocks, NWAP_SORT_WARPS * 32, 0, st>>>(src, dst, n, shift, c->d_sort_table, ntiles, tile);
        g_launches += 3;
        std::swap(src, dst);
    }
    const unsigned ublocks = (unsigned)std::min<long long>((n + 255) / 256, (long long)c->sm_count * 8);
    k_sort_unpack<<<ublocks, 256, 0, st>>>(src, n, (long long *)idx_out_dev, (signed char *)score_out_dev);
    g_launches++;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return NWAP_OK;
}

int nwap_score_range_compact(nwap_ctx *c, int64_t start, int64_t end, int8_t *out_dev, int threshold,
                             int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap, int64_t *count_host,
                             int32_t *degree_dev, nwap_stats *stats_host, int variant, void *stream)
{
    return score_sparse_common(c, start, end, out_dev, 1, threshold, 0.0, 0.0, idx_out_dev, score_out_dev, cap, count_host,
                               degree_dev, stats_host, variant, (cudaStream_t)stream);
}

int nwap_score_range_filter_normalized(nwap_ctx *c, int64_t start, int64_t end, int8_t *out_dev, double lo, double hi,
                                       int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap, int64_t *count_host,
                                       int32_t *degree_dev, nwap_stats *stats_host, int variant, void *stream)
{
    if (lo > hi) return fail(NWAP_EINVAL, "empty filter range: lo=%g > hi=%g", lo, hi);
    return score_sparse_common(c, start, end, out_dev, 2, 0, lo, hi, idx_out_dev, score_out_dev, cap, count_host,
                               degree_dev, stats_host, variant, (cudaStream_t)stream);
}

int nwap_filter_normalized(nwap_ctx *c, const int8_t *payload_dev, int64_t start, int64_t end, double lo, double hi,
                           int64_t *idx_out_dev, int8_t *score_out_dev, int64_t cap, int64_t *count_host,
                           int32_t *degree_dev, void *stream)
{
    if (!c) return fail(NWAP_EINVAL, "null context");
    if (lo > hi) return fail(NWAP_EINVAL, "empty filter range: lo=%g > hi=%g", lo, hi);
    nwap_keep_params kp;
    kp.threshold = 0; kp.lens = c->d_lens; kp.n = c->n; kp.start = start;
    nwap_fill_norm_bounds(kp, lo, hi, c->qmax);
    return compact_common(c, payload_dev, start, end, 1, kp, idx_out_dev, score_out_dev, cap, count_host, degree_dev,
                          (cudaStream_t)stream);
}

int nwap_hist_normalized(nwap_ctx *c, const int8_t *payload_dev, int64_t start, int64_t end,
                         uint64_t *counts_dev, void *stream)
{
    if (!c || !counts_dev) return fail(NWAP_EINVAL, "null argument");
    const int64_t P = nwap_num_edges(c);
    if (start < 0 || end > P || start > end) return fail(NWAP_EINVAL, "range [%lld, %lld) outside [0, %lld)", (long long)start, (long long)end, (long long)P);
    const int64_t count = end - start;
    if (count == 0) return NWAP_OK;
    if (!payload_dev) return fail(NWAP_EINVAL, "null payload");
    ON_DEVICE(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    nwap_keep_params kp;
    memset(&kp, 0, sizeof kp); kp.lens = c->d_lens; kp.n = c->n; kp.start = start;
    const int64_t runs = (count + NWAP_CMP_PER_THREAD - 1) / NWAP_CMP_PER_THREAD;
    if (c->qmax <= 100) {
        // joint (max length, score) bins: no per-edge division, 26 KB of shared memory at 24 symbols
        const size_t smem = sizeof(unsigned int) * (size_t)(256 + nwap_joint_mul(c->qmax)) * (size_t)(c->qmax + 1);
        const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / (smem + 1024)));
        CK(cudaFuncSetAttribute(k_hist_norm_joint_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int64_t wruns = (count + 15 + NWAP_HJ_RUN - 1) / NWAP_HJ_RUN;
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((wruns + 15) / 16, (int64_t)c->sm_count * per_sm));
        k_hist_norm_joint_w<<<(unsigned)blocks, 512, smem, st>>>(payload_dev, count, kp, (unsigned long long *)counts_dev, c->qmax);
        g_launches++;
        CK(cudaGetLastError());
        return NWAP_OK;
    }
    const size_t smem = sizeof(unsigned int) * NWAP_NHIST_SPAN;
    CK(cudaFuncSetAttribute(k_hist_normalized, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((runs + 511) / 512, (int64_t)c->sm_count * 2));
    k_hist_normalized<<<(unsigned)blocks, 512, smem, st>>>(payload_dev, count, kp, (unsigned long long *)counts_dev);
    g_launches++;
    CK(cudaGetLastError());
    return NWAP_OK;
}

int nwap_equal_work_bounds(const nwap_ctx *c, int parts, int64_t *bounds_out)
{
    if (!c || !bounds_out || parts < 1) return fail(NWAP_EINVAL, "bad argument");
    const int64_t n = c->n, P = n * (n - 1) / 2;
    const std::vector<int64_t> &pre = c->h_lenprefix;
    const std::vector<int64_t> &rowpref = c->h_rowpref;      // rowpref[r] = cells in rows < r
    const __int128 W = rowpref[n];
    bounds_out[0] = 0;
    for (int g = 1; g < parts; ++g) {
        const int64_t target = (int64_t)((W * g + parts - 1) / parts);
        // first row r with rowpref[r+1] >= target
        int64_t r = std::lower_bound(rowpref.begin() + 1, rowpref.end(), target) - (rowpref.begin() + 1);
        r = std::min<int64_t>(r, n - 2);
        const int64_t need = target - rowpref[r];
        int64_t col = r + 1;
        if (need > 0) {
            const int64_t lr = c->h_lens[r];
            const int64_t k = (need + lr - 1) / lr;
            col = std::lower_bound(pre.begin(), pre.end(), pre[r + 1] + k) - pre.begin();
        }
        int64_t idx = nwap_before_row(r, n) + (col - r - 1);
        idx = std::min(std::max(idx, bounds_out[g - 1]), P);
        bounds_out[g] = idx;
    }
    bounds_out[parts] = P;
    return NWAP_OK;
}

int nwap_rows_cols(int64_t n, const int64_t *idx_dev, int64_t count, int64_t *rows_dev, int64_t *cols_dev, void *stream)
{
    if (n < 2 || count < 0) return fail(NWAP_EINVAL, "bad argument");
    if (count == 0) return NWAP_OK;
    const int64_t blocks = std::min<int64_t>((count + 255) / 256, 4096);
    k_rows_cols<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, idx_dev, count, rows_dev, cols_dev);
    g_launches++;
    CK(cudaGetLastError());
    return NWAP_OK;
}

int nwap_probe(int device, int which, int iters, double *ipc_out, double *ms_out)
{
    if (which < 0 || which >= NWAP_PROBE_COUNT || iters < 1 || !ipc_out || !ms_out) return fail(NWAP_EINVAL, "bad argument");
    ON_DEVICE(device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    const int blocks = prop.multiProcessorCount;
    uint32_t *sink = nullptr;
    long long *cycles = nullptr;
    CK(cudaMalloc(&sink, 64));
    CK(cudaMalloc(&cycles, sizeof(long long) * blocks));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    typedef void (*probe_t)(int, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t *, long long *);
    static const probe_t table[NWAP_PROBE_COUNT] = {
        k_probe<0>, k_probe<1>, k_probe<2>, k_probe<3>, k_probe<4>, k_probe<5>, k_probe<6>, k_probe<7>,
        k_probe<8>, k_probe<9>, k_probe<10>, k_probe<11>, k_probe<12>, k_probe<13>, k_probe<14>, k_probe<15>,
        k_probe<16>, k_probe<17>, k_probe<18>, k_probe<19>, k_probe<20>, k_probe<21>, k_probe<22>, k_probe<23>,
        k_probe<24>, k_probe<25>, k_probe<26>, k_probe<27>, k_probe<28>, k_probe<29>};
    static const double per_step[NWAP_PROBE_COUNT] = {1, 1, 2, 1, 1, 1, 4, 4, 1, 2, 1, 2, 1, 2, 2, 2, 2, 2, 4, 5, 5, 2, 3, 2, 1, 2, 2, 4, 2, 2};
    for (int rep = 0; rep < 2; ++rep) {   // first launch warms up
        CK(cudaEventRecord(e0));
        table[which]<<<blocks, 512>>>(iters, 0x00030005u, 0xfffefffdu, 0x00070009u, 1u, sink, cycles);
        CK(cudaEventRecord(e1));
        g_launches++;
        CK(cudaGetLastError());
        CK(cudaEventSynchronize(e1));
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<long long> h(blocks);
    CK(cudaMemcpy(h.data(), cycles, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
    long long mx = 1;
    for (long long v : h) mx = std::max(mx, v);
    const double per_thread = per_step[which];           // instructions per chain step
    const double warp_instr = (double)iters * 16 * 8 * per_thread * (512 / 32);
    *ipc_out = warp_instr / (double)mx;
    *ms_out = ms;
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    cudaFree(sink); cudaFree(cycles);
    return NWAP_OK;
}

}  // extern "C"
