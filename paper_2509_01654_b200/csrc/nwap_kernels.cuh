// nwap_kernels.cuh -- the non-template sm_100a kernels around the tile kernel (nwap_tile.cuh): the generic
// one-thread-per-pair scorer, the dense-payload consumers, the key sort of the sparse-output mode and the
// instruction-issue probes.  Included by nwap.cu only (these are ordinary __global__ definitions).
#pragma once
#include "nwap_tile.cuh"

// ---------------------------------------------------------------------------
// Generic kernel: one thread per pair.  Rolling row in shared memory,
// transposed [column][thread] so lanes never conflict; similarity from a K x K
// int8 table in shared memory.  Any scheme, any q <= 255.
// ---------------------------------------------------------------------------
struct nwap_simple_params {
    const uint8_t *ids;
    const uint8_t *lens;
    int64_t n;
    int qpad;
    int qmax;
    int64_t start, end;
    int8_t *out;
    const int8_t *sim;     // (K, K) device
    int K;
    int gap;
    nwap_dev_stats *stats;
    int want_hist;
};

#define NWAP_SIMPLE_THREADS 128

__global__ void __launch_bounds__(NWAP_SIMPLE_THREADS)
k_score_simple(const nwap_simple_params p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int8_t *ssim = reinterpret_cast<int8_t *>(smem_raw);
    const int simbytes = (p.K * p.K + 15) & ~15;
    short *row = reinterpret_cast<short *>(smem_raw + simbytes);   // [(qmax+1)][THREADS]
    __shared__ unsigned int shist[256];
    __shared__ long long ssum, scount;
    __shared__ int smn, smx;

    const int tid = threadIdx.x;
    for (int i = tid; i < p.K * p.K; i += NWAP_SIMPLE_THREADS) ssim[i] = p.sim[i];
    for (int b = tid; b < 256; b += NWAP_SIMPLE_THREADS) shist[b] = 0;
    if (tid == 0) { ssum = 0; scount = 0; smn = 127; smx = -128; }
    __syncthreads();

    long long tsum = 0, tcnt = 0;
    int tmn = 127, tmx = -128;
    const int gap = p.gap;
    for (int64_t idx = p.start + (int64_t)blockIdx.x * NWAP_SIMPLE_THREADS + tid; idx < p.end;
         idx += (int64_t)gridDim.x * NWAP_SIMPLE_THREADS) {
        const int64_t r = nwap_row_of(idx, p.n);
        const int64_t c = nwap_col_of(idx, p.n, r);
        const uint8_t *a = p.ids + r * p.qpad;
        const uint8_t *b = p.ids + c * p.qpad;
        const int la = p.lens[r], lb = p.lens[c];
        for (int j = 0; j <= lb; ++j) row[j * NWAP_SIMPLE_THREADS + tid] = (short)(j * gap);
        for (int i = 1; i <= la; ++i) {
            const int8_t *srow = ssim + (int)a[i - 1] * p.K;
            int diag = row[tid];
            int left = i * gap;
            row[tid] = (short)left;
            for (int j = 1; j <= lb; ++j) {
                const int up = row[j * NWAP_SIMPLE_THREADS + tid];
                int v = diag + (int)srow[b[j - 1]];
                v = max(v, up + gap);
                v = max(v, left + gap);
                row[j * NWAP_SIMPLE_THREADS + tid] = (short)v;
                diag = up;
                left = v;
            }
        }
        const int s = row[lb * NWAP_SIMPLE_THREADS + tid];
        p.out[idx - p.start] = (int8_t)s;
        tsum += s; tcnt += 1; tmn = min(tmn, s); tmx = max(tmx, s);
        if (p.want_hist) atomicAdd(&shist[(s + 128) & 255], 1u);
    }
    atomicAdd(reinterpret_cast<unsigned long long *>(&ssum), (unsigned long long)tsum);
    atomicAdd(reinterpret_cast<unsigned long long *>(&scount), (unsigned long long)tcnt);
    atomicMin(&smn, tmn);
    atomicMax(&smx, tmx);
    __syncthreads();
    if (tid == 0 && scount > 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&p.stats->sum), (unsigned long long)ssum);
        atomicAdd(reinterpret_cast<unsigned long long *>(&p.stats->count), (unsigned long long)scount);
        atomicMin(&p.stats->mn, smn);
        atomicMax(&p.stats->mx, smx);
    }
    if (p.want_hist)
        for (int b = tid; b < 256; b += NWAP_SIMPLE_THREADS)
            if (shist[b]) atomicAdd(&p.stats->hist[b], (unsigned long long)shist[b]);
}

// ---------------------------------------------------------------------------
__global__ void k_init_stats(nwap_dev_stats *s, unsigned long long *counter)
{
    const int t = threadIdx.x;
    if (t < 256) s->hist[t] = 0;
    if (t == 0) { s->sum = 0; s->count = 0; s->mn = 127; s->mx = -128; if (counter) *counter = 0; }
}

// Dense payload -> statistics (HBM-bound: 1 byte read per edge).  The loop only feeds the 256-bin histogram
// (one shared-memory atomic per edge); sum, minimum and maximum are derived from the CTA's histogram at the end
// (thread t owns bin t, value t - 128), so the per-edge work is an extract and an atomic.
// hist_only: add the histogram only (the caller already holds sum / min / max / count from the scoring kernel).
__global__ void __launch_bounds__(256)
k_payload_stats(const int8_t *__restrict__ payload, int64_t count, nwap_dev_stats *stats, int hist_only)
{
    __shared__ unsigned int shist[256];
    __shared__ long long ssum;
    __shared__ int smn, smx;
    const int tid = threadIdx.x;
    shist[tid] = 0;
    if (tid == 0) { ssum = 0; smn = 127; smx = -128; }
    __syncthreads();
    // head bytes until 16-byte alignment, vector body, tail
    const uintptr_t addr = reinterpret_cast<uintptr_t>(payload);
    int64_t head = (int64_t)((16 - (addr & 15)) & 15);
    if (head > count) head = count;
    const int64_t nvec = (count - head) >> 4;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    if (gtid < head) atomicAdd(&shist[(int)payload[gtid] + 128], 1u);
    const uint4 *p4 = reinterpret_cast<const uint4 *>(payload + head);
    for (int64_t v = gtid; v < nvec; v += gstride) {
        const uint4 x = p4[v];
        const uint32_t w[4] = {x.x ^ 0x80808080u, x.y ^ 0x80808080u, x.z ^ 0x80808080u, x.w ^ 0x80808080u};   // bin = score + 128
#pragma unroll
        for (int k = 0; k < 16; ++k) atomicAdd(&shist[(w[k >> 2] >> (8 * (k & 3))) & 0xffu], 1u);
    }
    const int64_t tail0 = head + (nvec << 4);
    if (tail0 + gtid < count) atomicAdd(&shist[(int)payload[tail0 + gtid] + 128], 1u);
    __syncthreads();
    // thread t: bin t
    const unsigned int h = shist[tid];
    long long part = (long long)h * (long long)(tid - 128);
    int mn = h ? tid - 128 : 127, mx = h ? tid - 128 : -128;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        part += __shfl_xor_sync(0xffffffffu, part, o);
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((tid & 31) == 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&ssum), (unsigned long long)part);
        atomicMin(&smn, mn);
        atomicMax(&smx, mx);
    }
    if (h) atomicAdd(&stats->hist[tid], (unsigned long long)h);
    __syncthreads();
    if (tid == 0 && !hist_only) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&stats->sum), (unsigned long long)ssum);
        atomicMin(&stats->mn, smn);
        atomicMax(&stats->mx, smx);
        if (blockIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long *>(&stats->count), (unsigned long long)count);
    }
}

// ---------------------------------------------------------------------------
// Ordered compaction: count per block -> exclusive scan -> write.  The keep predicate is
//   MODE 0: raw score >= threshold
//   MODE 1: lo <= 100.0 * score / max(len_r, len_c) <= hi in IEEE double, exactly the
//           keep-mask of reference graph.py:96-98 (numpy float64 true division)
// Each thread owns 16 consecutive edges; for MODE 1 it recovers (r, c) of its first edge
// once (fp64 estimate + integer fix-up) and then walks the triangle.
// ---------------------------------------------------------------------------
#define NWAP_CMP_THREADS 256
#define NWAP_CMP_VEC 4                                              // 16-byte vectors per thread
#define NWAP_CMP_PER_THREAD (16 * NWAP_CMP_VEC)                     // 64 edges per thread
#define NWAP_CMP_BLOCK (NWAP_CMP_THREADS * NWAP_CMP_PER_THREAD)     // 16 KiB of the aligned window per block
#define NWAP_SCAN_PER 8                                             // block counts per thread of the scan
#define NWAP_SCAN_GROUP (1024 * NWAP_SCAN_PER)                      // block counts per scan CTA

// The payload slice is scanned through its 16-byte ALIGNED window: window byte w holds edge
// k = w - lead (lead = payload address & 15).  A thread owns 64 consecutive window bytes (four
// LDG.128); only the first and the last vector of the whole slice can straddle its ends and are
// assembled bytewise so nothing outside [payload, payload + count) is ever read.
__device__ __forceinline__ uint4 nwap_cmp_load(const int8_t *__restrict__ payload, int64_t count, int64_t k0)
{
    if (k0 >= 0 && k0 + 16 <= count) return *reinterpret_cast<const uint4 *>(payload + k0);
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int64_t k = k0 + j;
        if (k >= 0 && k < count) w[j >> 2] |= (uint32_t)(uint8_t)payload[k] << (8 * (j & 3));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// lens[c0 .. c0+63] as 16 packed words from 17 aligned 32-bit loads and byte permutes.  A thread's 64 edges of one
// row are 64 consecutive columns; fetching their lengths bytewise costs one L1 sector per lane per byte (lanes
// are 64 B apart), which made the normalised-weight kernels L1-bound.  Reads at most 3 bytes past c0+63: the
// device copy of lens is zero-padded by a whole strip.
__device__ __forceinline__ void nwap_load_lens64(const uint8_t *__restrict__ lens, int64_t c0, uint32_t (&V)[16])
{
    const uintptr_t a = reinterpret_cast<uintptr_t>(lens + c0);
    const uint32_t *p = reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3));
    const uint32_t sel = 0x3210u + 0x1111u * (uint32_t)(a & 3u);
    uint32_t w = __ldg(p);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t nx = __ldg(p + j + 1);
        V[j] = __byte_perm(w, nx, sel);
        w = nx;
    }
}

// Rows of a compaction block (16 KiB of consecutive edges): almost always one or two, so one thread recovers
// the first row (fp64 estimate + integer fix-up) and everyone else places itself by two comparisons.
struct nwap_block_rows {
    long long r0;          // row of the block's first live edge (-1: block holds no live edge)
    long long next1;       // edge offset (relative to payload[0]) at which row r0 + 1 begins
    long long next2;       // ... and row r0 + 2
};

__device__ __forceinline__ void nwap_block_rows_init(nwap_block_rows *br, const nwap_keep_params &kp, int64_t k_block,
                                                     int64_t count);
__device__ __forceinline__ void nwap_block_rows_sync(nwap_block_rows *br, const nwap_keep_params &kp, int64_t k_block,
                                                     int64_t count)
{
    nwap_block_rows_init(br, kp, k_block, count);
    __syncthreads();
}
__device__ __forceinline__ void nwap_block_rows_init(nwap_block_rows *br, const nwap_keep_params &kp, int64_t k_block,
                                                     int64_t count)
{
    if (threadIdx.x == 0) {
        const int64_t kb = max(k_block, (int64_t)0);
        br->r0 = -1; br->next1 = br->next2 = 0;
        if (kb < count) {
            const int64_t r = nwap_row_of(kp.start + kb, kp.n);
            br->r0 = r;
            br->next1 = nwap_before_row(r + 1, kp.n) - kp.start;
            br->next2 = nwap_before_row(min(r + 2, kp.n - 1), kp.n) - kp.start;
        }
    }
}

// MODE 1, phase A: load the thread's 64 window bytes and mark the CANDIDATES from the payload alone -- a score outside
// [gmin, gmax] (the loosest bounds over all lengths) cannot be kept whatever the word lengths are.  Needs nothing but
// the payload and two scalars, so a block whose threads find no candidate is done without any index recovery, bounds
// table or barrier (selective filters: almost every block).
__device__ __forceinline__ unsigned long long nwap_window_load(const int8_t *__restrict__ payload, int64_t count,
                                                               int64_t k_first, uint4 (&vec)[NWAP_CMP_VEC])
{
    if (k_first >= count || k_first + NWAP_CMP_PER_THREAD <= 0) {
#pragma unroll
        for (int v = 0; v < NWAP_CMP_VEC; ++v) vec[v] = make_uint4(0u, 0u, 0u, 0u);
        return 0;
    }
#pragma unroll
    for (int v = 0; v < NWAP_CMP_VEC; ++v) vec[v] = nwap_cmp_load(payload, count, k_first + 16 * v);
    unsigned long long valid = ~0ull;                            // validity mask of this thread's 64 window bytes
    if (k_first < 0) valid &= ~0ull << (int)(-k_first);
    if (k_first + NWAP_CMP_PER_THREAD > count) valid &= ~0ull >> (int)(k_first + NWAP_CMP_PER_THREAD - count);
    return valid;
}
__device__ __forceinline__ unsigned long long nwap_cand_bits(const nwap_keep_params &kp, const uint4 (&vec)[NWAP_CMP_VEC],
                                                             unsigned long long valid)
{
    if (valid == 0 || kp.gmin > kp.gmax) return 0;
    unsigned long long cand = 0;
    {
        const uint32_t Tlo = (uint32_t)(kp.gmin + 128);                 // gmin >= -128
        const uint32_t lo_rep = (Tlo & 0x7fu) * 0x01010101u;
        const bool lo_th = (Tlo & 0x80u) != 0;
        const bool all_lo = kp.gmin <= -128;
        const bool has_hi = kp.gmax < 127;
        const uint32_t Thi = (uint32_t)(kp.gmax + 1 + 128);              // scores >= gmax + 1 are out
        const uint32_t hi_rep = (Thi & 0x7fu) * 0x01010101u;
        const bool hi_th = (Thi & 0x80u) != 0;
#pragma unroll
        for (int v = 0; v < NWAP_CMP_VEC; ++v) {
            const uint32_t w[4] = {vec[v].x, vec[v].y, vec[v].z, vec[v].w};
            unsigned b16 = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                unsigned ok = all_lo ? 0xfu : nwap_ge_bits4(w[q], lo_rep, lo_th);
                if (has_hi) ok &= ~nwap_ge_bits4(w[q], hi_rep, hi_th);
                b16 |= ok << (4 * q);
            }
            cand |= (unsigned long long)b16 << (16 * v);
        }
        cand &= valid;
    }
    return cand;
}

// MODE 1, phase B: the exact keep-mask of the candidates -- lo <= 100.0*score/max(len_r, len_c) <= hi (graph.py:96-98)
// through the per-length score bounds in shared memory; (r, c) walks the triangle.
__device__ __forceinline__ unsigned long long nwap_keep_eval(int64_t count, int64_t k_first, const nwap_keep_params &kp,
                                                             const uint4 (&vec)[NWAP_CMP_VEC], unsigned long long cand,
                                                             unsigned long long valid, const short2 *bounds,
                                                             const short2 *rbounds, const nwap_block_rows *br)
{
    unsigned long long bits = 0;
    if (cand == 0) return 0;
    const int64_t kb = max(k_first, (int64_t)0);
    const int64_t ke = min(k_first + (int64_t)NWAP_CMP_PER_THREAD, count) - 1;       // last live edge of this thread
    // the block's one or two rows were recovered once (nwap_block_rows_init); a thread places itself by comparisons
    int64_t r = -1;
    if (br->r0 >= 0) {
        if (ke < br->next1) r = br->r0;
        else if (kb >= br->next1 && ke < br->next2) r = br->r0 + 1;
    }
    const bool one_row = r >= 0;
    if (!one_row) r = nwap_row_of(kp.start + kb, kp.n);
    if (one_row && __popcll(cand) <= 8) {
        // all live edges of this thread lie in row r: its own length tightens the candidate bounds (m >= len_r),
        // and the few survivors fetch their column length one byte each
        const int lr1 = (int)kp.lens[r];
        const short2 rb = rbounds[lr1];
        const int64_t c0 = r + 1 + (kp.start + k_first - nwap_before_row(r, kp.n));  // column of window byte 0 (may precede the row for masked bytes)
        unsigned long long rest = cand;
        while (rest) {
            const int e = __ffsll((long long)rest) - 1;
            rest &= rest - 1;
            const uint4 q = vec[e >> 4];
            const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
            const int sc = (int)(int8_t)((w4[(e >> 2) & 3] >> (8 * (e & 3))) & 0xffu);
            if (sc < (int)rb.x || sc > (int)rb.y) continue;
            const short2 b = bounds[max(lr1, (int)kp.lens[c0 + e])];
            if (sc >= (int)b.x && sc <= (int)b.y) bits |= 1ull << e;
        }
        return bits;
    }
    int64_t c = nwap_col_of(kp.start + kb, kp.n, r);
    int lr = (int)kp.lens[r];
    if (valid == ~0ull && c + NWAP_CMP_PER_THREAD <= kp.n) {
        // the usual case: 64 live edges of one row = 64 consecutive columns
        uint32_t L[16];
        nwap_load_lens64(kp.lens, c, L);
#pragma unroll
        for (int v = 0; v < NWAP_CMP_VEC; ++v) {
            const uint32_t w[4] = {vec[v].x, vec[v].y, vec[v].z, vec[v].w};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int e = 16 * v + j;
                if ((cand >> e) & 1ull) {
                    const int sc = (int)(int8_t)((w[j >> 2] >> (8 * (j & 3))) & 0xffu);
                    const int lc = (int)((L[e >> 2] >> (8 * (e & 3))) & 0xffu);
                    const short2 b = bounds[max(lr, lc)];
                    if (sc >= (int)b.x && sc <= (int)b.y) bits |= 1ull << e;
                }
            }
        }
        return bits;
    }
#pragma unroll
    for (int v = 0; v < NWAP_CMP_VEC; ++v) {
        const uint32_t w[4] = {vec[v].x, vec[v].y, vec[v].z, vec[v].w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int e = 16 * v + j;
            if ((valid >> e) & 1ull) {
                const int sc = (int)(int8_t)((w[j >> 2] >> (8 * (j & 3))) & 0xffu);
                const short2 b = bounds[max(lr, (int)kp.lens[c])];
                if (sc >= (int)b.x && sc <= (int)b.y) bits |= 1ull << e;
                if (++c == kp.n) { ++r; c = r + 1; lr = (int)kp.lens[min(r, kp.n - 1)]; }
            }
        }
    }
    return bits;
}

template <int MODE>
__device__ __forceinline__ unsigned long long nwap_keep_bits(const int8_t *__restrict__ payload, int64_t count,
                                                             int64_t k_first, const nwap_keep_params &kp,
                                                             uint4 (&vec)[NWAP_CMP_VEC], const short2 *bounds,
                                                             const short2 *rbounds = nullptr,
                                                             nwap_block_rows *br = nullptr)
{
    unsigned long long bits = 0;
    if (MODE == 0) {
        const unsigned long long valid = nwap_window_load(payload, count, k_first, vec);
        if (valid == 0) return 0;
        const int t = kp.threshold;
        if (t > 127) return 0;
        if (t <= -128) return valid;
        const uint32_t T = (uint32_t)(t + 128);
        const uint32_t tl_rep = (T & 0x7fu) * 0x01010101u;
        const bool th = (T & 0x80u) != 0;
#pragma unroll
        for (int v = 0; v < NWAP_CMP_VEC; ++v) {
            const uint32_t w[4] = {vec[v].x, vec[v].y, vec[v].z, vec[v].w};
            unsigned b16 = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) b16 |= nwap_ge_bits4(w[q], tl_rep, th) << (4 * q);
            bits |= (unsigned long long)b16 << (16 * v);
        }
        return bits & valid;
    }
    // MODE 1: the payload loads are issued first; the block's rows are recovered by thread 0 while they are in flight
    // (the barrier inside nwap_block_rows_sync), then candidates from the payload alone, then the exact test
    const unsigned long long valid1 = nwap_window_load(payload, count, k_first, vec);
    nwap_block_rows_sync(br, kp, k_first - (int64_t)threadIdx.x * NWAP_CMP_PER_THREAD, count);
    const unsigned long long cand = nwap_cand_bits(kp, vec, valid1);
    if (cand == 0) return 0;
    return nwap_keep_eval(count, k_first, kp, vec, cand, valid1, bounds, rbounds, br);
}

// first window byte of (block, thread), as an edge offset relative to payload[0] (may be negative)
__device__ __forceinline__ int64_t nwap_cmp_first(const int8_t *payload)
{
    const int64_t lead = (int64_t)(reinterpret_cast<uintptr_t>(payload) & 15u);
    return ((int64_t)blockIdx.x * NWAP_CMP_THREADS + threadIdx.x) * NWAP_CMP_PER_THREAD - lead;
}

template <int MODE>
__global__ void __launch_bounds__(NWAP_CMP_THREADS)
k_compact_count(const int8_t *__restrict__ payload, int64_t count, const nwap_keep_params kp, long long *block_counts,
                unsigned long long *group_totals)
{
    // MODE 1: the per-length score bounds live in a 2 KB device table (kp.dtab: [0, 256) per m, [256, 512) per row
    // length) read through L1 by the few threads that hold a candidate.  (Staging them in shared memory from the
    // kernel parameters cost a 32-way serialised constant load per warp and a barrier per 16 KB block: 1.2 TB/s.)
    __shared__ nwap_block_rows brows;
    uint4 vec[NWAP_CMP_VEC];
    const int kept = __popcll(nwap_keep_bits<MODE>(payload, count, nwap_cmp_first(payload), kp, vec, kp.dtab, kp.dtab + 256, &brows));
    __shared__ int wsum[NWAP_CMP_THREADS / 32];
    const int wkept = __reduce_add_sync(0xffffffffu, kept);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = wkept;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < NWAP_CMP_THREADS / 32; ++w) tot += wsum[w];
        block_counts[blockIdx.x] = tot;
        if (tot) atomicAdd(&group_totals[blockIdx.x / NWAP_SCAN_GROUP], (unsigned long long)tot);   // kept edges are rare
    }
}

// Exclusive scan of block_counts (in place), one CTA per group of NWAP_SCAN_GROUP counts: the group's base is
// the sum of the totals of the groups before it (accumulated by k_compact_count), then a local scan with 8
// consecutive counts per thread.  CTA 0 also writes the grand total.
__global__ void __launch_bounds__(1024)
k_compact_scan(long long *block_counts, int64_t nblocks, const unsigned long long *group_totals, int64_t ngroups,
               long long *total_out)
{
    __shared__ long long wtot[32];
    __shared__ long long base_s;
    // base = sum of group_totals[0 .. blockIdx.x)  (and the grand total in CTA 0)
    long long part = 0, all = 0;
    for (int64_t g = threadIdx.x; g < ngroups; g += 1024) {
        const long long v = (long long)group_totals[g];
        if (g < (int64_t)blockIdx.x) part += v;
        all += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { part += __shfl_xor_sync(0xffffffffu, part, o); all += __shfl_xor_sync(0xffffffffu, all, o); }
    if ((threadIdx.x & 31) == 0) wtot[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) { long long b = 0; for (int w = 0; w < 32; ++w) b += wtot[w]; base_s = b; }
    __syncthreads();
    if (blockIdx.x == 0) {
        __syncthreads();
        if ((threadIdx.x & 31) == 0) wtot[threadIdx.x >> 5] = all;
        __syncthreads();
        if (threadIdx.x == 0) { long long t = 0; for (int w = 0; w < 32; ++w) t += wtot[w]; *total_out = t; }
        __syncthreads();
    }
    const int64_t i0 = (int64_t)blockIdx.x * NWAP_SCAN_GROUP + (int64_t)threadIdx.x * NWAP_SCAN_PER;
    long long v[NWAP_SCAN_PER];
    long long tsum = 0;
#pragma unroll
    for (int k = 0; k < NWAP_SCAN_PER; ++k) {
        v[k] = i0 + k < nblocks ? block_counts[i0 + k] : 0;
        tsum += v[k];
    }
    long long x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) wtot[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        long long w = wtot[threadIdx.x], ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, ws, o);
            if (threadIdx.x >= o) ws += y;
        }
        wtot[threadIdx.x] = ws - w;      // exclusive warp offsets
    }
    __syncthreads();
    long long run = base_s + wtot[threadIdx.x >> 5] + (x - tsum);
#pragma unroll
    for (int k = 0; k < NWAP_SCAN_PER; ++k) {
        if (i0 + k < nblocks) block_counts[i0 + k] = run;
        run += v[k];
    }
}

// Blocks that keep nothing (the usual case: C5 keeps 2e-5 of the edges) return before touching the
// payload again, so the second pass costs one read of the block offsets plus the few non-empty blocks.
template <int MODE>
__global__ void __launch_bounds__(NWAP_CMP_THREADS)
k_compact_write(const int8_t *__restrict__ payload, int64_t count, const nwap_keep_params kp,
                const long long *block_offsets, const long long *total, int64_t nblocks,
                int64_t *idx_out, int8_t *score_out, int64_t cap, int *degree)
{
    const long long off0 = block_offsets[blockIdx.x];
    const long long off1 = (int64_t)blockIdx.x + 1 < nblocks ? block_offsets[blockIdx.x + 1] : *total;
    if (off1 == off0) return;
    const int64_t k_first = nwap_cmp_first(payload);
    __shared__ nwap_block_rows brows;
    uint4 vec[NWAP_CMP_VEC];
    const unsigned long long bits = nwap_keep_bits<MODE>(payload, count, k_first, kp, vec, kp.dtab, kp.dtab + 256, &brows);
    const int kept = __popcll(bits);
    // exclusive scan of `kept` over the block
    __shared__ int wtot[NWAP_CMP_THREADS / 32];
    int x = kept;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) wtot[threadIdx.x >> 5] = x;
    __syncthreads();
    int woff = 0;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) woff += wtot[w];
    int64_t pos = off0 + woff + (x - kept);
    unsigned long long rest = bits;
    while (rest) {
        const int e = __ffsll((long long)rest) - 1;
        rest &= rest - 1;
        const int64_t idx = kp.start + k_first + e;
        if (pos < cap) {
            const uint4 q = vec[e >> 4];
            const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
            idx_out[pos] = idx;
            score_out[pos] = (int8_t)((w4[(e >> 2) & 3] >> (8 * (e & 3))) & 0xffu);
        }
        if (degree) {
            const int64_t r = nwap_row_of(idx, kp.n);
            const int64_t c = nwap_col_of(idx, kp.n, r);
            atomicAdd(&degree[r], 1);
            atomicAdd(&degree[c], 1);
        }
        ++pos;
    }
}

// ---------------------------------------------------------------------------
// Order restoration for the sparse-output mode: LSD radix sort (8 bits per pass) of the 64-bit keys
// (linear index << 8 | score byte).  One warp owns a contiguous tile of keys (a multiple of 32, at least
// NWAP_SORT_TILE, grown so that there are at most 65,536 tiles):
//   k_sort_hist     per-tile digit counts -> table[digit][tile]
//   k_sort_scan     exclusive scan of the table in (digit, tile) order, one CTA
//   k_sort_scatter  the warp walks its tile 32 keys at a time; equal digits are ranked in lane order with
//                   __match_any_sync, so the pass is stable
//   k_sort_unpack   keys -> (int64 index, int8 score)
// Kept edges are few (C5 keeps 2e-5 of 1.8e11), so this is a fraction of a millisecond per pass.
// ---------------------------------------------------------------------------
#define NWAP_SORT_TILE 2048
#define NWAP_SORT_WARPS 8

__global__ void __launch_bounds__(NWAP_SORT_WARPS * 32)
k_sort_hist(const unsigned long long *__restrict__ keys, long long n, int shift, unsigned int *table, long long ntiles,
            long long tile_size)
{
    __shared__ unsigned int cnt[NWAP_SORT_WARPS][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long tile = (long long)blockIdx.x * NWAP_SORT_WARPS + warp;
    for (int d = lane; d < 256; d += 32) cnt[warp][d] = 0;
    __syncwarp();
    if (tile < ntiles) {
        const long long k0 = tile * tile_size, k1 = min(k0 + tile_size, n);
        for (long long k = k0 + lane; k < k1; k += 32) atomicAdd(&cnt[warp][(unsigned)(keys[k] >> shift) & 255u], 1u);
        __syncwarp();
        for (int d = lane; d < 256; d += 32) table[(long long)d * ntiles + tile] = cnt[warp][d];
    }
}

__global__ void __launch_bounds__(1024)
k_sort_scan(unsigned int *table, long long count)
{
    __shared__ unsigned int wtot[32];
    __shared__ unsigned int carry;          // sum of all trips before the current one
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < count; base += 1024 * 8) {
        const long long i0 = base + (long long)threadIdx.x * 8;
        unsigned int v[8], tsum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) { v[k] = i0 + k < count ? table[i0 + k] : 0u; tsum += v[k]; }
        unsigned int x = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const unsigned int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
        if (lane == 31) wtot[warp] = x;
        __syncthreads();
        const unsigned int c = carry;       // read by everyone before it is advanced below
        unsigned int trip_total = 0;
        if (warp == 0) {
            const unsigned int w = wtot[lane];
            unsigned int ws = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const unsigned int y = __shfl_up_sync(0xffffffffu, ws, o); if (lane >= o) ws += y; }
            wtot[lane] = ws - w;            // exclusive warp offsets
            trip_total = ws;                // lane 31: the trip's total
        }
        __syncthreads();
        if (warp == 0 && lane == 31) carry = c + trip_total;
        unsigned int run = c + wtot[warp] + (x - tsum);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (i0 + k < count) table[i0 + k] = run;
            run += v[k];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NWAP_SORT_WARPS * 32)
k_sort_scatter(const unsigned long long *__restrict__ in, unsigned long long *__restrict__ out, long long n, int shift,
               const unsigned int *__restrict__ table, long long ntiles, long long tile_size)
{
    __shared__ unsigned int off[NWAP_SORT_WARPS][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long tile = (long long)blockIdx.x * NWAP_SORT_WARPS + warp;
    if (tile >= ntiles) return;
    for (int d = lane; d < 256; d += 32) off[warp][d] = table[(long long)d * ntiles + tile];
    __syncwarp();
    const long long k0 = tile * tile_size, k1 = min(k0 + tile_size, n);
    const unsigned lt = (1u << lane) - 1u;
    for (long long kb = k0; kb < k1; kb += 32) {
        const long long k = kb + lane;
        const bool valid = k < k1;
        const unsigned long long key = valid ? in[k] : 0ull;
        const unsigned d = valid ? (unsigned)(key >> shift) & 255u : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        unsigned int basepos = 0;
        if (valid) basepos = off[warp][d];
        __syncwarp();
        if (valid) {
            out[basepos + rank] = key;
            if (rank == 0) off[warp][d] = basepos + __popc(peers);
        }
        __syncwarp();
    }
}

__global__ void k_sort_unpack(const unsigned long long *keys, long long n, long long *idx_out, signed char *score_out)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        idx_out[i] = (long long)(k >> 8);
        score_out[i] = (signed char)(k & 0xffu);
    }
}

// ---------------------------------------------------------------------------
// Normalised histogram (reference store.py:352-366, normalized=True): bin of
// floor(100*score / max(len_r, len_c)) in exact integer arithmetic, values in
// [-12800, 12700] -> 25,501 bins.  Counts are privatised per CTA in shared memory
// (25,501 x u32 = 100 KB) and flushed once.
// ---------------------------------------------------------------------------
#define NWAP_NHIST_OFFSET (-12800)
#define NWAP_NHIST_SPAN 25501

__global__ void __launch_bounds__(512)
k_hist_normalized(const int8_t *__restrict__ payload, int64_t count, const nwap_keep_params kp,
                  unsigned long long *counts)
{
    extern __shared__ unsigned int sbins[];
    for (int b = threadIdx.x; b < NWAP_NHIST_SPAN; b += blockDim.x) sbins[b] = 0;
    __syncthreads();
    // The slice is read through its 16-byte aligned window, 64 edges (four LDG.128) per thread per trip, as in
    // the compaction scan.  floor(100*s / m) is taken from an IEEE single division: |100*s| <= 12800 and
    // m <= 255 are exact floats, an integral quotient is exact, and a non-integral one is at least 1/255 away
    // from the next integer (relative 3e-7 > 2^-24), so rounding never reaches it; checked exhaustively on the
    // host for all 256 x 255 (s, m) in tests/test_core_emul.py.
    const int64_t lead = (int64_t)(reinterpret_cast<uintptr_t>(payload) & 15u);
    const int64_t runs = (lead + count + NWAP_CMP_PER_THREAD - 1) / NWAP_CMP_PER_THREAD;
    for (int64_t run = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; run < runs; run += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k_first = run * NWAP_CMP_PER_THREAD - lead;
        const int64_t kb = max(k_first, (int64_t)0);
        if (kb >= count) continue;
        int64_t r = nwap_row_of(kp.start + kb, kp.n);
        int64_t c = nwap_col_of(kp.start + kb, kp.n, r);
        int lr = (int)kp.lens[r];
        if (k_first >= 0 && k_first + NWAP_CMP_PER_THREAD <= count && c + NWAP_CMP_PER_THREAD <= kp.n) {
            // the usual case: 64 live edges of one row = 64 consecutive columns (vector loads for both streams)
            uint32_t L[16];
            nwap_load_lens64(kp.lens, c, L);
#pragma unroll
            for (int v = 0; v < NWAP_CMP_VEC; ++v) {
                const uint4 q4 = *reinterpret_cast<const uint4 *>(payload + k_first + 16 * v);
                const uint32_t w[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int e = 16 * v + j;
                    const int m = max(lr, (int)((L[e >> 2] >> (8 * (e & 3))) & 0xffu));
                    const int num = 100 * (int)(int8_t)((w[j >> 2] >> (8 * (j & 3))) & 0xffu);
                    atomicAdd(&sbins[nwap_floor_div_small(num, m) - NWAP_NHIST_OFFSET], 1u);
                }
            }
            continue;
        }
#pragma unroll
        for (int v = 0; v < NWAP_CMP_VEC; ++v) {
            const int64_t k0 = k_first + 16 * v;
            if (k0 + 16 <= 0 || k0 >= count) continue;
            const uint4 q4 = nwap_cmp_load(payload, count, k0);
            const uint32_t w[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int64_t k = k0 + j;
                if (k >= 0 && k < count) {
                    const int m = max(lr, (int)kp.lens[c]);
                    const int num = 100 * (int)(int8_t)((w[j >> 2] >> (8 * (j & 3))) & 0xffu);
                    const int q = nwap_floor_div_small(num, m);
                    atomicAdd(&sbins[q - NWAP_NHIST_OFFSET], 1u);
                    if (++c == kp.n) { ++r; c = r + 1; lr = (int)kp.lens[min(r, kp.n - 1)]; }
                }
            }
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NWAP_NHIST_SPAN; b += blockDim.x)
        if (sbins[b]) atomicAdd(&counts[b], (unsigned long long)sbins[b]);
}

// The same histogram without per-edge arithmetic: count the JOINT key (m, score), m = max(len_r, len_c), in
// (mmax + 1) x 256 shared-memory bins -- per edge one byte-permute and one shared atomic, the per-4-edges maximum
// of the lengths as byte-parallel integer ops -- and map each occupied (m, score) bin to floor(100*score / m) ONCE
// per CTA at the end, in exact integer arithmetic (store.py:357-361).  Needs mmax <= 127 (byte-parallel max on
// 7-bit lengths) and (mmax + 1) KB of shared memory; longer words use k_hist_normalized.
// swizzle multiplier of the joint histogram: the largest odd j in {9, 5, 3, 1} with mmax * j < 256
__host__ __device__ inline int nwap_joint_mul(int mmax) { return mmax <= 28 ? 9 : mmax <= 51 ? 5 : mmax <= 85 ? 3 : 1; }
__device__ __forceinline__ uint32_t nwap_bytemax7(uint32_t a, uint32_t b)        // per-byte max, all bytes < 128
{
    const uint32_t ge = (((a | 0x80808080u) - b) >> 7) & 0x01010101u;             // 1 where a >= b
    const uint32_t mask = ge * 0xffu;
    return (a & mask) | (b & ~mask);
}

// prmt.b32, default mode: selector nibble k < 8 copies byte k of {a, b}; nibble 8|k replicates the msb of byte k
__device__ __forceinline__ uint32_t nwap_prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// Work distribution.  The L1 / shared pipe is this kernel's bound, and in its first version (one thread = 64 consecutive
// edges, as in the compaction scan: 1.23 TB/s, ncu 99 %) most wavefronts were not the atomics: four LDG.128 that lie 64
// bytes apart between neighbouring lanes (16 cache lines per warp instruction) plus seventeen LDG.32 of lengths with the
// same stride: 64 + 272 wavefronts per 2048 edges against ~130 for the atomics.  Here a WARP owns 2048 consecutive
// window bytes and lane l takes the 16-byte vectors 32k + l (k = 0..3):
// every payload instruction covers 512 contiguous bytes (16 sectors), and the 16 lengths of a vector come from the two
// aligned LDG.128 that hold them (16 sectors each across the warp).  Order does not matter
// for a histogram.  (r, c) is recovered once per warp run; a run that crosses a row end or the ends of the slice
// (one in ~300 at 600,000 words) takes the per-edge walk.
#define NWAP_HJ_RUN 2048
__global__ void __launch_bounds__(512)
k_hist_norm_joint_w(const int8_t *__restrict__ payload, int64_t count, const nwap_keep_params kp,
                    unsigned long long *counts, int mmax)
{
    extern __shared__ unsigned int jbins[];              // [(mmax + 1) * JS]
    const int jmul = nwap_joint_mul(mmax), JS = 256 + jmul;
    const int nb = (mmax + 1) * JS;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) jbins[b] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t lead = (int64_t)(reinterpret_cast<uintptr_t>(payload) & 15u);
    const int64_t runs = (lead + count + NWAP_HJ_RUN - 1) / NWAP_HJ_RUN;
    // a warp owns a CONTIGUOUS range of runs, so the row is recovered once (fp64 estimate + fix-up: ~150 warp
    // instructions, a fifth of the kernel when done per run) and then walked
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t rpw = (runs + nwarps - 1) / nwarps;
    const int64_t run_lo = warp0 * rpw, run_hi = min(runs, run_lo + rpw);
    int64_t r = -1, row0 = 0, row_end = 0;                       // row of the current edge: global edges [row0, row_end)
    for (int64_t run = run_lo; run < run_hi; ++run) {
        const int64_t k_run = run * NWAP_HJ_RUN - lead;          // edge offset of the run's window byte 0 (may be negative)
        const int64_t kb = max(k_run, (int64_t)0);
        const int64_t ke = min(k_run + (int64_t)NWAP_HJ_RUN, count) - 1;   // last live edge of the run
        if (kb > ke) continue;
        if (r < 0) {
            r = nwap_row_of(kp.start + kb, kp.n);                // the same value in every lane
            row0 = nwap_before_row(r, kp.n);
            row_end = row0 + (kp.n - 1 - r);
        }
        while (kp.start + kb >= row_end) { ++r; row0 = row_end; row_end += kp.n - 1 - r; }
        const bool whole = k_run >= 0 && k_run + NWAP_HJ_RUN <= count && kp.start + ke < row_end;
        if (whole) {
            const int lr = (int)kp.lens[r];
            const uint32_t lr4 = (uint32_t)lr * 0x01010101u;
            const int64_t c_run = r + 1 + (kp.start + k_run - row0);     // column of the run's window byte 0
#pragma unroll
            for (int k = 0; k < NWAP_HJ_RUN / 512; ++k) {
                const int off = 512 * k + 16 * lane;
                const uint4 q4 = *reinterpret_cast<const uint4 *>(payload + k_run + off);
                // lengths of columns c_run + off .. + 15: the two aligned 16-byte vectors that hold them (across the
                // warp: 2 x 16 sectors instead of 5 x 16 with word loads), realigned by whole words (uniform: every
                // lane of the run has the same misalignment) and then by bytes
                const uintptr_t a = reinterpret_cast<uintptr_t>(kp.lens + c_run + off);
                const uint4 *lp = reinterpret_cast<const uint4 *>(a & ~uintptr_t(15));
                const uint4 v0 = __ldg(lp), v1 = __ldg(lp + 1);
                const uint32_t sel = 0x3210u + 0x1111u * (uint32_t)(a & 3u);
                uint32_t lw[5];
                switch ((int)((a >> 2) & 3u)) {
                case 0: lw[0] = v0.x; lw[1] = v0.y; lw[2] = v0.z; lw[3] = v0.w; lw[4] = v1.x; break;
                case 1: lw[0] = v0.y; lw[1] = v0.z; lw[2] = v0.w; lw[3] = v1.x; lw[4] = v1.y; break;
                case 2: lw[0] = v0.z; lw[1] = v0.w; lw[2] = v1.x; lw[3] = v1.y; lw[4] = v1.z; break;
                default: lw[0] = v0.w; lw[1] = v1.x; lw[2] = v1.y; lw[3] = v1.z; lw[4] = v1.w; break;
                }
                const uint32_t w[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t x = w[q] ^ 0x80808080u;                       // score + 128 per byte
                    const uint32_t m4 = nwap_bytemax7(__byte_perm(lw[q], lw[q + 1], sel), lr4);
                    const uint32_t s4 = m4 * (uint32_t)jmul;                     // swizzle term per byte (mmax * jmul < 256)
                    atomicAdd(&jbins[nwap_prmt(x, m4, 0xcc40u) + nwap_prmt(s4, 0u, 0x4440u)], 1u);
                    atomicAdd(&jbins[nwap_prmt(x, m4, 0xdd51u) + nwap_prmt(s4, 0u, 0x4441u)], 1u);
                    atomicAdd(&jbins[nwap_prmt(x, m4, 0xee62u) + nwap_prmt(s4, 0u, 0x4442u)], 1u);
                    atomicAdd(&jbins[nwap_prmt(x, m4, 0xff73u) + nwap_prmt(s4, 0u, 0x4443u)], 1u);
                }
            }
            continue;
        }
        // the run crosses a row end or an end of the slice: lane l walks edges kb + l, kb + l + 32, ...
        for (int64_t k = kb + lane; k <= ke; k += 32) {
            const int64_t rr = nwap_row_of(kp.start + k, kp.n);
            const int64_t cc = nwap_col_of(kp.start + k, kp.n, rr);
            const int m = max((int)kp.lens[rr], (int)kp.lens[cc]);
            const int sb = (int)payload[k] + 128;
            atomicAdd(&jbins[m * JS + sb], 1u);
        }
    }
    __syncthreads();
    for (int b = JS + threadIdx.x; b < nb; b += blockDim.x) {   // m = 0 never occurs (every word has >= 1 symbol)
        const unsigned int h = jbins[b];
        if (h) {
            const int m = b / JS, sb = b - m * JS;
            if (sb > 255) continue;                                         // padding words of the swizzled layout
            const int num = 100 * (sb - 128);
            int qv = num / m;
            if (num % m != 0 && num < 0) --qv;                          // floor division
            atomicAdd(&counts[qv - NWAP_NHIST_OFFSET], (unsigned long long)h);
        }
    }
}

__global__ void k_rows_cols(int64_t n, const int64_t *idx, int64_t count, int64_t *rows, int64_t *cols)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = nwap_row_of(idx[i], n);
        rows[i] = r;
        cols[i] = nwap_col_of(idx[i], n, r);
    }
}

// ---------------------------------------------------------------------------
// Instruction-issue probes: 8 independent chains per thread, unrolled 16x, every
// operation an `asm volatile` so nothing is folded.  See NWAP_PROBE_* in nwap.h.
// ---------------------------------------------------------------------------
#define NWAP_OP3(name, x, a, b) asm volatile(name " %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b))
#define NWAP_OP2(name, x, a) asm volatile(name " %0, %0, %1;" : "+r"(x) : "r"(a))
__device__ __forceinline__ void nwap_p_viaddmin(uint32_t &x, uint32_t a, uint32_t c)
{ asm volatile("{.reg .b32 t; add.u16x2 t, %0, %1; min.u16x2 %0, t, %2;}" : "+r"(x) : "r"(a), "r"(c)); }
__device__ __forceinline__ void nwap_p_vimax3(uint32_t &x, uint32_t a, uint32_t c)
{ asm volatile("{.reg .b32 t; max.s16x2 t, %0, %1; max.s16x2 %0, t, %2;}" : "+r"(x) : "r"(a), "r"(c)); }
__device__ __forceinline__ void nwap_p_imad(uint32_t &x, uint32_t a, uint32_t c)
{ asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(c)); }

template <int WHICH>
__global__ void __launch_bounds__(512)
k_probe(int iters, uint32_t a, uint32_t b, uint32_t c, uint32_t one, uint32_t *sink, long long *cycles)
{
    uint32_t x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { x[k] = a + threadIdx.x * 8 + k; y[k] = b ^ (threadIdx.x + k); }
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (WHICH == 0) nwap_p_viaddmin(x[k], b, c);
                else if (WHICH == 1) nwap_p_vimax3(x[k], b, y[k]);
                else if (WHICH == 2) { NWAP_OP2("max.s16x2", x[k], y[k]); NWAP_OP2("max.s16x2", y[k], x[k]); }   // dependent pair: ptxas cannot fuse it into VIMNMX3
                else if (WHICH == 3) nwap_p_imad(x[k], a, b);
                else if (WHICH == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"(b), "r"(y[k]));
                else if (WHICH == 5) asm volatile("{.reg .b32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[k]) : "r"(y[k]), "r"(b));   // one IADD3
                else if (WHICH == 6) {                                    // 2 DPX + 2 IMAD cell
                    uint32_t e = a; nwap_p_viaddmin(e, y[k], 0x00010001u);
                    nwap_p_imad(e, b, x[k]);
                    nwap_p_vimax3(x[k], e, y[k]);
                    y[k] = x[k]; nwap_p_imad(y[k], one, c);
                } else if (WHICH == 7) {                                  // 3 DPX/ALU + 1 IMAD cell
                    uint32_t e = a; nwap_p_viaddmin(e, y[k], 0x00010001u);
                    nwap_p_imad(e, b, x[k]);
                    asm volatile("{.reg .b32 t; add.s16x2 t, %0, %1; max.s16x2 %0, t, %2;}" : "+r"(y[k]) : "r"(c), "r"(e));
                    NWAP_OP2("max.s16x2", x[k], y[k]);
                }
                else if (WHICH == 8) NWAP_OP2("add.u16x2", x[k], y[k]);
                else if (WHICH == 9) { NWAP_OP2("min.u16x2", x[k], y[k]); NWAP_OP2("min.u16x2", y[k], x[k]); }
                else if (WHICH == 10) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(a), "r"(b));
                else if (WHICH == 11) { NWAP_OP2("max.f16x2", x[k], y[k]); NWAP_OP2("max.f16x2", y[k], x[k]); }
                else if (WHICH == 12) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(y[k]), "r"(b));
                else if (WHICH == 13) { nwap_p_vimax3(x[k], b, c); NWAP_OP2("add.u32", y[k], a); }          // DPX + IADD
                else if (WHICH == 14) { nwap_p_vimax3(x[k], b, c); NWAP_OP2("max.s16x2", y[k], a); }        // DPX + VIMNMX2
                else if (WHICH == 15) { nwap_p_imad(x[k], a, b); NWAP_OP2("add.u32", y[k], a); }            // IMAD + IADD
                else if (WHICH == 16) { nwap_p_imad(x[k], a, b); asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(y[k]) : "r"(a), "r"(b)); }
                else if (WHICH == 17) { nwap_p_vimax3(x[k], b, c); nwap_p_imad(y[k], a, b); }               // DPX + IMAD
                else if (WHICH == 18) {                                   // cell with IADD for up+u: 2 DPX + IMAD + IADD
                    uint32_t e = a; nwap_p_viaddmin(e, y[k], 0x00010001u);
                    nwap_p_imad(e, b, x[k]);
                    nwap_p_vimax3(x[k], e, y[k]);
                    y[k] = x[k]; NWAP_OP2("add.u32", y[k], c);
                } else if (WHICH == 19) {                                 // cell with 2-input max: DPX + 2 IMAD + 2 VIMNMX2
                    uint32_t e = a; nwap_p_viaddmin(e, y[k], 0x00010001u);
                    nwap_p_imad(e, b, x[k]);
                    NWAP_OP2("max.s16x2", x[k], e); NWAP_OP2("max.s16x2", x[k], y[k]);
                    y[k] = x[k]; nwap_p_imad(y[k], one, c);
                } else if (WHICH == 20) {                                 // cell: xor + min2 + IMAD + VIMNMX3 + IMAD
                    uint32_t e = a; NWAP_OP2("xor.b32", e, y[k]); NWAP_OP2("min.u16x2", e, one);
                    nwap_p_imad(e, b, x[k]);
                    nwap_p_vimax3(x[k], e, y[k]);
                    y[k] = x[k]; nwap_p_imad(y[k], one, c);
                } else if (WHICH == 21) { nwap_p_viaddmin(x[k], b, c); nwap_p_vimax3(y[k], b, c); }         // two DPX kinds
                else if (WHICH == 23) {                                   // dependent add pair (cannot be merged)
                    NWAP_OP2("add.u32", x[k], y[k]); NWAP_OP2("add.u32", y[k], x[k]);
                } else if (WHICH == 24) asm volatile("set.ne.f16x2.f16x2 %0, %0, %1;" : "+r"(x[k]) : "r"(y[k]));   // HSET2.BF
                else if (WHICH == 25) {                                   // HSET2 + DPX
                    asm volatile("set.ne.f16x2.f16x2 %0, %0, %1;" : "+r"(x[k]) : "r"(b));
                    nwap_p_vimax3(y[k], b, c);
                } else if (WHICH == 26) {                                 // dependent adds + DPX, 1:1
                    uint32_t &w = x[(k + 4) & 7];
                    if (k < 4) { NWAP_OP2("add.u32", x[k], w); nwap_p_vimax3(y[k], b, c); NWAP_OP2("add.u32", w, x[k]); nwap_p_vimax3(y[k + 4], b, c); }
                } else if (WHICH == 27) {                                 // fp16-compare cell: HSET2 + HFMA2 + DPX + add
                    uint32_t e = a; asm volatile("set.ne.f16x2.f16x2 %0, %0, %1;" : "+r"(e) : "r"(y[k]));
                    asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(e) : "r"(b), "r"(x[k]));
                    nwap_p_vimax3(x[k], e, y[k]);
                    y[k] = x[k]; NWAP_OP2("add.u32", y[k], c);
                } else if (WHICH == 28) {                                 // HSET2 + IMAD
                    asm volatile("set.ne.f16x2.f16x2 %0, %0, %1;" : "+r"(x[k]) : "r"(b));
                    nwap_p_imad(y[k], a, b);
                } else if (WHICH == 29) {                                 // dependent adds + IMAD, 1:1
                    uint32_t &w = x[(k + 4) & 7];
                    if (k < 4) { NWAP_OP2("add.u32", x[k], w); nwap_p_imad(y[k], a, b); NWAP_OP2("add.u32", w, x[k]); nwap_p_imad(y[k + 4], a, b); }
                }
                else if (WHICH == 22) {                                   // symmetric-potential cell: 2 DPX + IADD3
                    uint32_t e = a; nwap_p_viaddmin(e, x[k], c);
                    asm volatile("{.reg .b32 t; sub.u32 t, %1, %0; add.u32 %0, t, %2;}" : "+r"(e) : "r"(x[k]), "r"(b));
                    nwap_p_vimax3(x[k], e, y[k]);
                }
            }
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= x[k] ^ y[k];
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}
