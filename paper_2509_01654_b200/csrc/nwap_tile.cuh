// nwap_tile.cuh -- the hot kernel of the all-pairs NW scoring path (k_score_tiles) and what it shares with the
// consumers.  Templates and inline device code only: included by every tiles_*.cu instantiation unit.
// (kernel inventory of the whole library:)
//
//   k_score_tiles<FLAVOR,QMAX>  the hot kernel: persistent 10-warp CTAs (two per SM) over (strip, band-group)
//                               work units; per unit the strip's 5120 columns are counting-sorted by word
//                               length in shared memory, warps pull 64-column chunks longest-first (so the
//                               warps of a CTA sit in neighbouring length-specialised bodies), each lane
//                               scores 2 pairs per register (s16x2 DPX); one length dispatch per chunk, the
//                               body owning the loop over the band's 16 rows; results are staged in shared
//                               memory at their ORIGINAL column and flushed as coalesced 16-byte stores.
//                               Replaces reference engine.py:176-195 (_score_range) with
//                               triangle.py:93-112 folded in (one index recovery per row).
//   k_score_simple              one thread per pair, int32 cells, K x K similarity table:
//                               any scheme (overrides), any q <= 255.  Generic path and the
//                               independent second implementation used for cross-checks.
//   k_payload_stats             sum/min/max/count/hist of a dense payload (store.py:342-381 raw).
//   k_compact_*                 ordered threshold compaction + degree counts (graph.py:97-101).
//   k_rows_cols                 triangle.py:93-112 exposed for parity tests.
//   k_probe<W>                  instruction-issue probes for the integer roofline.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "nwap_core.cuh"
#include "nwap_index.cuh"

#ifndef NWAP_LBSTEP
#define NWAP_LBSTEP 1
#endif
#ifndef NWAP_MINB
#define NWAP_MINB 2               // resident CTAs/SM the register allocator must allow
#endif
#ifndef NWAP_UNITS_PER_SLOT
#define NWAP_UNITS_PER_SLOT 48
#endif
#define NWAP_WARPS (NWAP_THREADS / 32)
#define NWAP_MAXLEN_FAST 32              // register-resident row limit
#ifndef NWAP_WIDE_FROM
#define NWAP_WIDE_FROM 24                // uniform schemes: vocabularies whose longest word exceeds this run the wide build
#endif

struct nwap_dev_stats {                   // same layout as nwap_stats
    long long sum;
    long long count;
    int mn;
    int mx;
    unsigned long long hist[256];
};

// ---------------------------------------------------------------------------
// Keep predicate of the threshold compaction / normalised-weight filter (graph.py:91-101), shared by the
// dense-payload consumers (k_compact_*) and the tile kernel's sparse-output mode.
// ---------------------------------------------------------------------------
struct nwap_keep_params {
    int threshold;           // MODE 0
    const uint8_t *lens;     // MODE 1
    int64_t n;
    int64_t start;           // linear index of payload[0]
    // MODE 1: for every m = max(len_r, len_c) the scores s with lo <= 100.0*s/m <= hi form an interval
    // [smin[m], smax[m]] (the quotient is monotonic in s).  The host fills the table by evaluating the
    // reference's IEEE-double expression (graph.py:96-98) for all 256 x 255 (s, m), so the device test is
    // two integer compares and exactly the reference's keep-mask; an empty interval is smin > smax.
    int8_t smin[256], smax[256];
    int gmin, gmax;          // MODE 1: loosest bounds over all lengths (gmin > gmax: nothing can be kept)
    // MODE 1: loosest bounds over the lengths m >= l (up to the longest word): what a score in a row whose word has
    // l symbols must satisfy whatever the column is, since m = max(len_r, len_c) >= len_r.  Empty: rmin > rmax.
    int8_t rmin[256], rmax[256];
    const short2 *dtab;      // MODE 1: the same bounds on the device: [m] = (smin, smax), [256 + l] = (rmin, rmax)
};

// host side of the table above
inline void nwap_fill_norm_bounds(nwap_keep_params &kp, double lo, double hi, int qmax = 255)
{
    for (int m = 0; m < 256; ++m) {
        int first = 1, last = 0;                     // empty
        bool any = false;
        for (int sc = -128; sc <= 127 && m > 0; ++sc) {
            const double w = (100.0 * (double)sc) / (double)m;
            if (w >= lo && w <= hi) { if (!any) first = sc; last = sc; any = true; }
        }
        kp.smin[m] = (int8_t)first;
        kp.smax[m] = (int8_t)last;
    }
    kp.gmin = 127; kp.gmax = -128;
    for (int m = 1; m < 256; ++m)
        if (kp.smin[m] <= kp.smax[m]) { kp.gmin = kp.gmin < kp.smin[m] ? kp.gmin : kp.smin[m]; kp.gmax = kp.gmax > kp.smax[m] ? kp.gmax : kp.smax[m]; }
    int lo_s = 127, hi_s = -128;                      // running loosest bounds over m in [l, qmax]
    for (int l = 255; l >= 0; --l) {
        if (l >= 1 && l <= qmax && kp.smin[l] <= kp.smax[l]) {
            lo_s = lo_s < kp.smin[l] ? lo_s : kp.smin[l];
            hi_s = hi_s > kp.smax[l] ? hi_s : kp.smax[l];
        }
        kp.rmin[l] = (int8_t)(lo_s <= hi_s ? lo_s : 1);
        kp.rmax[l] = (int8_t)(lo_s <= hi_s ? hi_s : 0);
    }
}

// MODE 0: bit j of the result = (signed byte j of the 4 words >= threshold), 4 bytes per SWAR step.
// x = w ^ 0x80808080 orders the bytes as unsigned; T = threshold + 128 in [0, 255].
__device__ __forceinline__ unsigned nwap_ge_bits4(uint32_t w, uint32_t tl_rep, bool th)
{
    const uint32_t x = w ^ 0x80808080u;
    const uint32_t d = ((x & 0x7f7f7f7fu) | 0x80808080u) - tl_rep;     // bit 7 of a byte: low 7 bits >= low 7 bits of T
    const uint32_t m = (th ? (x & d) : (x | d)) & 0x80808080u;
    return (((m >> 7) * 0x01020408u) >> 24) & 0xfu;
}

// Sparse-output mode of the tile kernel (BASELINE north_star: "the int8 edge writer, with optional
// score-threshold compaction"): kept edges leave the kernel as unordered 64-bit keys
// (linear index << 8 | score byte) appended through one global counter; a radix sort of the keys
// restores index order afterwards (k_sort_*).  The dense payload need not exist at all.
struct nwap_sparse_out {
    int mode;                       // 0: off, 1: raw score >= threshold, 2: normalised-weight bounds (graph.py:96-98)
    int threshold;                  // mode 1
    int gmin, gmax;                 // mode 2: loosest score bounds over all lengths (candidates)
    const short2 *bounds;           // mode 2: device table of 256 per-length (smin, smax)
    unsigned long long *keys;       // device, `cap` entries
    long long cap;
    unsigned long long *count;      // device counter (may exceed cap: the excess is dropped, the host reports it)
    int *degree;                    // device (n,) or NULL: +1 at both endpoints of every kept edge
};

struct nwap_tile_params {
    const uint8_t *ids;      // (n, qpad) uint8
    const uint8_t *lens;     // (n padded to strips) uint8, zero beyond n
    int64_t n;
    int qpad;
    int64_t start, end;      // linear range
    int64_t r_first, r_last; // rows holding start and end-1
    int64_t c_start, c_end;  // column of start, column of end-1 (inclusive)
    int8_t *out;             // out[k - start]
    nwap_scheme_consts sc;
    nwap_unit_space us;
    int64_t unit_begin;      // absolute id of the first unit of this launch
    int64_t unit_count;
    unsigned long long *unit_counter;
    nwap_dev_stats *stats;
    int want_hist;                 // unused by the tile kernel (see k_payload_stats); kept for the generic kernel's twin struct
    const nwap_ov_row *ov_table;   // sparse-override mode: (ov_K) rows on the device, else NULL
    int ov_K;                      // alphabet size K of the override / dense table
    const uint8_t *etab;           // dense-table mode (FLAVOR 3): K x K table of M - sim on the device, else NULL
    int tab2_lmax;                 // FLAVOR 3: > 0 = the row-pair profiles fit shared memory (rows per profile), see nwap_chunk_rows_tab2
    nwap_sparse_out sparse;        // CMP instantiations only
};

struct alignas(16) nwap_row_meta {
    // first 16 bytes: everything the fast row path needs
    int la;            // row word length, 0 = row not in this launch / no valid column in this strip
    uint32_t symend;   // (uint32)(-8 * la): the matrix-row loop's counter, which runs up to zero (nwap_chunk_rows_fast2)
    uint32_t ala2;     // (alpha * la) * 65537: the row potential, packed for both halves
    int rowadj;        // smem byte index of (column offset 0): rr*PITCH + skew - clo_off
    int clo_off;       // first valid column, relative to the strip
    int seglen;        // number of valid columns in this strip for this row
    int64_t g0;        // out-relative byte offset of the segment
};
// (global address of the row's segment) & 15: the staged row is skewed so shared and global addresses agree mod 16
template <int PITCH>
__device__ __forceinline__ int nwap_meta_skew(const nwap_row_meta &m, int rr) { return m.rowadj - rr * PITCH + m.clo_off; }

// ---------------------------------------------------------------------------
// shared memory carve-up of k_score_tiles
// ---------------------------------------------------------------------------
#define NWAP_OV_MAXK 128               // largest alphabet the sparse-override table holds in shared memory
#define NWAP_TAB_MAXK 256              // largest alphabet of the table-driven cell: K x K bytes of dynamic shared memory
                                       // (64 KB at 256 symbols: one CTA per SM; two up to ~100 symbols)
template <int MODE> struct nwap_sym_of { typedef nwap_sym2 type; };
template <> struct nwap_sym_of<1> { typedef nwap_sym8 type; };

// MODE 0: uniform scheme, 1: sparse overrides (per-symbol correction rows), 2: dense table (K x K bytes of M - sim)
// MAXLEN: longest word the instantiation accepts (32, or 64 for the block-wise wide build)
// CW: strip width in columns.  NWAP_TAB_CW = NWAP_C / 2 gives the table-driven flavour half-width strips (output stage
// and sorted-column arrays 48 KB smaller: room for two CTAs per SM next to the row-pair profiles) -- measured: -5.6 %
// while its 168 registers keep it at one CTA per SM anyway, so the default is the full width.
#ifndef NWAP_TAB_CW
#define NWAP_TAB_CW NWAP_C
#endif
template <int MODE, int MAXLEN = NWAP_MAXLEN_FAST, int CW = (MODE == 2 ? NWAP_TAB_CW : NWAP_C)>
struct nwap_tile_smem_t {
    static constexpr int C = CW;                 // columns per strip
    static constexpr int PITCH = CW + 16;        // bytes per staged output row (multiple of 16)
    static_assert(CW % (4 * NWAP_THREADS) == 0 && CW <= NWAP_C && NWAP_C % CW == 0, "strip width");
    alignas(16) uint8_t out[NWAP_R * PITCH];
    typedef typename nwap_sym_of<MODE>::type sym_t;
    alignas(16) sym_t rowsym[NWAP_R][MAXLEN + 1];                // {a*65537, H'[i+1][0] (, override row)} per matrix row
    // first staged record of row rr.  The 8-byte records of a row END at slot MAXLEN (so that the matrix-row loop of
    // the fast2 family can count a negative offset up to zero against a warp-uniform base); override rows start at 0.
    static constexpr bool END_ALIGNED = MODE != 1;
    __device__ __forceinline__ const sym_t *syms(int rr, int la) const { return rowsym[rr] + (END_ALIGNED ? MAXLEN - la : 0); }
    __device__ __forceinline__ sym_t *syms(int rr, int la) { return rowsym[rr] + (END_ALIGNED ? MAXLEN - la : 0); }
    alignas(16) nwap_ov_part ov[MODE == 1 ? NWAP_OV_MAXK : 1];      // per-symbol partner table (sparse-override mode)
    alignas(16) nwap_row_meta meta[NWAP_R + 1];                     // one readable record past the band (row prefetch)
    uint16_t cols[CW];            // strip-relative column offsets, sorted by length desc
    uint8_t clen[CW];             // their lengths
    int bins[NWAP_WARPS][MAXLEN + 2];
    short2 kbounds[256];          // sparse-output mode, normalised filter: per-length score bounds
    unsigned long long unit;
    long long sum;
    long long count;
    int mn, mx;
    int ncols;                    // sorted columns of the unit: [0, nclean) by length, longest first; [nclean, ncols) unsorted
    int nclean;
    int next_chunk;
    uint8_t t2order[NWAP_R];      // FLAVOR 3, second shape: the band's rows in order of length (rows are paired by length)
    // dense-table mode: K x K bytes of M - sim.  LAST member: the launch sizes the dynamic shared memory to the
    // alphabet actually used (nwap_tile_smem_bytes), so that tables of up to ~100 symbols leave room for two CTAs per SM
    alignas(16) uint8_t etab[MODE == 2 ? NWAP_TAB_MAXK * NWAP_TAB_MAXK : 16];
};

typedef nwap_tile_smem_t<0> nwap_tile_smem;

__device__ __forceinline__ uint32_t nwap_byte_of(const uint32_t *w, int j)
{
    return (w[j >> 2] >> (8 * (j & 3))) & 0xffu;
}

// Column codes of the lane's two words for matrix columns 0..N-1 (nwap_pack_negb_f).  FLAVOR 1: byte permutes only --
// {A0 A1 B0 B1} per two columns, then {A0 ff B0 ff} and {A1 ff B1 ff}: three PRMT per two columns.
template <int FLAVOR, int N, int QW>
__device__ __forceinline__ void nwap_unpack_cols(const uint32_t (&w0)[QW], const uint32_t (&w1)[QW], uint32_t (&nb)[N])
{
    if (FLAVOR == 1) {
#pragma unroll
        for (int j = 0; j < N; j += 2) {
            const uint32_t t = __byte_perm(w0[j >> 2], w1[j >> 2], (j & 2) ? 0x7632u : 0x5410u);
            nb[j] = __byte_perm(t, 0xffffffffu, 0x4240u);
            if (j + 1 < N) nb[j + 1] = __byte_perm(t, 0xffffffffu, 0x4341u);
        }
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j) nb[j] = nwap_pack_negb_f<FLAVOR>(nwap_byte_of(w0, j), nwap_byte_of(w1, j));
    }
}

// Statistics are kept packed: t = H' + row potential + column potential has halves
// score + BIAS, so min/max are one VIMNMX.S16x2 each for both pairs and the byte to store
// is simply the low byte of each half (BIAS is a multiple of 256).
struct nwap_lane_stats {
    uint32_t mn2, mx2;      // packed running min / max of (score + BIAS)
    long long sum;          // sum of scores
    int count;              // valid pairs
};

// One lane's two columns of a 64-column chunk.
struct nwap_lane_cols {
    uint32_t off0, off1;    // strip-relative column offsets (0xffff = no column)
    int l0, l1;             // word lengths
    uint32_t kpos2;         // column potentials, packed (BIAS stays in: halves of t are score + BIAS)
    uint32_t keep_v;        // per-half mask: 0xffff where the word has length LB
    uint32_t keep_1;        // per-half mask: 0xffff where the word has length LB-1 (else LB-2 in mixmode 2)
};

__device__ __forceinline__ nwap_lane_cols nwap_make_lane_cols(uint32_t off0, uint32_t off1, int l0, int l1, int LB,
                                                              const nwap_scheme_consts &sc)
{
    nwap_lane_cols c;
    c.off0 = off0; c.off1 = off1; c.l0 = l0; c.l1 = l1;
    c.kpos2 = (uint32_t)(sc.beta * l0) + ((uint32_t)(sc.beta * l1) << 16);
    c.keep_v = (l0 == LB ? 0xffffu : 0u) | (l1 == LB ? 0xffff0000u : 0u);
    c.keep_1 = (l0 == LB - 1 ? 0xffffu : 0u) | (l1 == LB - 1 ? 0xffff0000u : 0u);
    return c;
}

// Per-chunk packed accumulators of t (<= 2 * 16 rows: no overflow of either half-sum).
struct nwap_chunk_acc { uint32_t acc, acc_hi; int rows_fast; };

// Score fix-up, staging store and statistics of one packed result (shared by all lengths).
template <class SM>
__device__ __forceinline__ void nwap_emit(SM &sm, const nwap_row_meta &m, uint32_t ala2, int adj, uint32_t v,
                                          const nwap_lane_cols &c, bool fast, int want_hist,
                                          nwap_lane_stats &ls, nwap_chunk_acc &ca)
{
    const uint32_t t = v + ala2 + c.kpos2;          // halves: score + BIAS (never negative)
    const uint32_t thi = t >> 16;
    if (fast) {
        sm.out[adj + (int)c.off0] = (uint8_t)t;
        sm.out[adj + (int)c.off1] = (uint8_t)thi;
        ls.mn2 = __vmins2(ls.mn2, t);
        ls.mx2 = __vmaxs2(ls.mx2, t);
        ca.acc += t;
        ca.acc_hi += thi;
        ++ca.rows_fast;
    } else {
        const uint32_t clo = (uint32_t)m.clo_off;
        const uint32_t seg = (uint32_t)m.seglen;
        const int s0 = (int)(t & 0xffffu) - (int)NWAP_BIAS;
        const int s1 = (int)thi - (int)NWAP_BIAS;
        if (c.off0 - clo < seg) {
            sm.out[adj + (int)c.off0] = (uint8_t)(int8_t)s0;
            ls.sum += s0; ls.count += 1;
            ls.mn2 = __vmins2(ls.mn2, (ls.mn2 & 0xffff0000u) | (t & 0xffffu));
            ls.mx2 = __vmaxs2(ls.mx2, (ls.mx2 & 0xffff0000u) | (t & 0xffffu));
        }
        if (c.off1 - clo < seg) {
            sm.out[adj + (int)c.off1] = (uint8_t)(int8_t)s1;
            ls.sum += s1; ls.count += 1;
            ls.mn2 = __vmins2(ls.mn2, (ls.mn2 & 0xffffu) | (t & 0xffff0000u));
            ls.mx2 = __vmaxs2(ls.mx2, (ls.mx2 & 0xffffu) | (t & 0xffff0000u));
        }
    }
}

__device__ __forceinline__ void nwap_close_chunk(nwap_lane_stats &ls, const nwap_chunk_acc &ca)
{
    if (ca.rows_fast) {
        // acc = sum(lo) + 65536 * sum(hi) (mod 2^32), acc_hi = sum(hi): both sums < 2^19
        const uint32_t sum_lo = ca.acc - (ca.acc_hi << 16);
        ls.sum += (long long)sum_lo + (long long)ca.acc_hi - 2ll * ca.rows_fast * (long long)NWAP_BIAS;
        ls.count += 2 * ca.rows_fast;
    }
}

// mixmode 1/2: pick the final cell of each half among the last three columns (bitwise selects)
__device__ __forceinline__ uint32_t nwap_merge3(uint32_t v, uint32_t vm1, uint32_t vm2, const nwap_lane_cols &c)
{
    const uint32_t t = (vm1 & c.keep_1) | (vm2 & ~c.keep_1);
    return (v & c.keep_v) | (t & ~c.keep_v);
}

struct nwap_true { __device__ constexpr operator bool() const { return true; } };
struct nwap_false { __device__ constexpr operator bool() const { return false; } };

// The only length-specialised code: the DP of one row word at register width LB.  Returns the
// final cells for words of length LB (v) and LB-1 (vm1) -- all a sorted chunk normally
// contains; `deep` (a chunk spanning three or more lengths: the long and short tails of a
// strip) selects per lane among all columns.
template <int LB, int FLAVOR>
__device__ __forceinline__ void nwap_dp_word_sel(const nwap_sym2 *sym, int la, const uint32_t *nb, uint32_t (&P)[LB + 1],
                                                 const nwap_scheme_consts &sc, const nwap_ov_part *)
{
    nwap_dp_word<LB, FLAVOR>(sym, la, nb, P, sc);
}
template <int LB, int FLAVOR>
__device__ __forceinline__ void nwap_dp_word_sel(const nwap_sym8 *sym, int la, const uint32_t *nb, uint32_t (&P)[LB + 1],
                                                 const nwap_scheme_consts &sc, const nwap_ov_part *parts)
{
    nwap_dp_word_ov<LB, FLAVOR>(sym, la, nb, P, sc, parts);
}

template <int LB, int FLAVOR, class SYM>
__device__ __forceinline__ void nwap_row_dp(const SYM *sym, const nwap_ov_part *ovtab, int la, const uint32_t *nb,
                                            int l0, int l1, const nwap_scheme_consts &sc, uint32_t &v, uint32_t &vm1,
                                            uint32_t &vm2, bool deep)
{
    uint32_t P[LB + 1];
    nwap_dp_word_sel<LB, FLAVOR>(sym, la, nb, P, sc, ovtab);
    v = P[LB];
    vm1 = P[LB >= 2 ? LB - 1 : LB];
    vm2 = P[LB >= 3 ? LB - 2 : LB];
    if (deep) {
        uint32_t lo = v & 0xffffu, hi = v & 0xffff0000u;
#pragma unroll
        for (int j = 1; j < LB; ++j) {
            if (j == l0) lo = P[j] & 0xffffu;
            if (j == l1) hi = P[j] & 0xffff0000u;
        }
        v = lo | hi;
    }
}

#define NWAP_CASES_1_32                                                                        \
    NWAP_CASE(1) NWAP_CASE(2) NWAP_CASE(3) NWAP_CASE(4) NWAP_CASE(5) NWAP_CASE(6) NWAP_CASE(7) NWAP_CASE(8)         \
    NWAP_CASE(9) NWAP_CASE(10) NWAP_CASE(11) NWAP_CASE(12) NWAP_CASE(13) NWAP_CASE(14) NWAP_CASE(15) NWAP_CASE(16)  \
    NWAP_CASE(17) NWAP_CASE(18) NWAP_CASE(19) NWAP_CASE(20) NWAP_CASE(21) NWAP_CASE(22) NWAP_CASE(23) NWAP_CASE(24) \
    NWAP_CASE(25) NWAP_CASE(26) NWAP_CASE(27) NWAP_CASE(28) NWAP_CASE(29) NWAP_CASE(30) NWAP_CASE(31) NWAP_CASE(32)

// One chunk (64 sorted columns, 2 per lane) against every staged row of the band.
// mixmode: 0 = every lane of the warp has both words of length LB; 1 = some are LB-1 (the
// usual case at a bucket boundary of the sorted strip); 2 = anything.  fast: the chunk is full
// and every staged row is valid over the whole column window, so no per-lane range checks are
// needed (the overwhelmingly common case).  All warp-uniform.
template <int FLAVOR, int QMAX, int QW, class SM>
__device__ __forceinline__ void nwap_run_chunk(int LB, SM &sm, const nwap_scheme_consts &sc,
                                               const uint32_t (&w0)[QW], const uint32_t (&w1)[QW],
                                               const nwap_lane_cols &c, int mixmode, bool fast,
                                               int want_hist, nwap_lane_stats &ls)
{
    uint32_t nb[QMAX];
    nwap_unpack_cols<FLAVOR, QMAX, QW>(w0, w1, nb);
    nwap_chunk_acc ca; ca.acc = 0; ca.acc_hi = 0; ca.rows_fast = 0;
    const bool deep = mixmode > 2;
    const int l0 = c.l0, l1 = c.l1;
#pragma unroll 1
    for (int rr = 0; rr < NWAP_R; ++rr) {
        const nwap_row_meta &m = sm.meta[rr];
        const int la = m.la;
        if (la == 0) continue;                       // uniform across the CTA
        const typename SM::sym_t *sym = sm.syms(rr, la);
        uint32_t v = 0, vm1 = 0, vm2 = 0;
#define NWAP_CASE(n)                                                                                       \
    case n:                                                                                                \
        if (n <= QMAX) nwap_row_dp<(n <= QMAX ? n : 1), FLAVOR>(sym, sm.ov, la, nb, l0, l1, sc, v, vm1, vm2, deep); \
        break;
        switch (LB) { NWAP_CASES_1_32 default: break; }
#undef NWAP_CASE
        if (mixmode == 1 || mixmode == 2) v = nwap_merge3(v, vm1, vm2, c);
        nwap_emit(sm, m, m.ala2, m.rowadj, v, c, fast, want_hist, ls, ca);
    }
    nwap_close_chunk(ls, ca);
}


// Dense-table chunks (FLAVOR 3): per-row dispatch with the shared epilogue; the lane's column symbols are kept
// as byte offsets (two registers per matrix column) for the table loads of nwap_dp_row_tab.
template <int LB>
__device__ __forceinline__ void nwap_row_dp_tab(const nwap_sym2 *sym, int la, const uint32_t *c0, const uint32_t *c1,
                                                int l0, int l1, const nwap_scheme_consts &sc, const uint8_t *etab,
                                                uint32_t &v, uint32_t &vm1, uint32_t &vm2, bool deep)
{
    uint32_t P[LB + 1];
    nwap_dp_word_tab<LB>(sym, la, c0, c1, P, sc, etab);
    v = P[LB];
    vm1 = P[LB >= 2 ? LB - 1 : LB];
    vm2 = P[LB >= 3 ? LB - 2 : LB];
    if (deep) {
        uint32_t lo = v & 0xffffu, hi = v & 0xffff0000u;
#pragma unroll
        for (int j = 1; j < LB; ++j) {
            if (j == l0) lo = P[j] & 0xffffu;
            if (j == l1) hi = P[j] & 0xffff0000u;
        }
        v = lo | hi;
    }
}

// one length dispatch per chunk; the body owns the loop over the band's rows (as the hoisted uniform-scheme bodies)
template <int LB, class SM>
__device__ __forceinline__ void nwap_chunk_rows_tab(SM &sm, const nwap_scheme_consts &sc, const uint32_t *c0,
                                                    const uint32_t *c1, const nwap_lane_cols &c, int mixmode, bool fast,
                                                    int want_hist, nwap_lane_stats &ls, nwap_chunk_acc &ca)
{
    const bool deep = mixmode > 2;
#pragma unroll 1
    for (int rr = 0; rr < NWAP_R; ++rr) {
        const nwap_row_meta &m = sm.meta[rr];
        const int la = m.la;
        if (la == 0) continue;
        uint32_t v, vm1, vm2;
        nwap_row_dp_tab<LB>(reinterpret_cast<const nwap_sym2 *>(sm.syms(rr, la)), la, c0, c1, c.l0, c.l1, sc, sm.etab,
                            v, vm1, vm2, deep);
        if (mixmode == 1 || mixmode == 2) v = nwap_merge3(v, vm1, vm2, c);
        nwap_emit(sm, m, m.ala2, m.rowadj, v, c, fast, want_hist, ls, ca);
    }
}

template <int QMAX, int QW, class SM>
__device__ __forceinline__ void nwap_run_chunk_tab(int LB, SM &sm, const nwap_scheme_consts &sc,
                                                   const uint32_t (&w0)[QW], const uint32_t (&w1)[QW],
                                                   const nwap_lane_cols &c, int mixmode, bool fast,
                                                   int want_hist, nwap_lane_stats &ls)
{
    uint32_t c0[QMAX], c1[QMAX];
#pragma unroll
    for (int j = 0; j < QMAX; ++j) { c0[j] = nwap_byte_of(w0, j); c1[j] = nwap_byte_of(w1, j); }
    nwap_chunk_acc ca; ca.acc = 0; ca.acc_hi = 0; ca.rows_fast = 0;
#define NWAP_CASE(n)                                                                                       \
    case n:                                                                                                \
        if (n <= QMAX) nwap_chunk_rows_tab<(n <= QMAX ? n : 1)>(sm, sc, c0, c1, c, mixmode, fast, want_hist, ls, ca); \
        break;
    switch (LB) { NWAP_CASES_1_32 default: break; }
#undef NWAP_CASE
    nwap_close_chunk(ls, ca);
}

// NWAP_HOIST=1 (default): the length dispatch is done once per chunk and each length body owns the
// whole row loop with the emit inlined.  With 4-warp CTAs this lost 13-18 % to instruction-cache
// misses (profiles/r01e); with 10-warp CTAs it gains 3-4 % (profiles/r01h_ab_big_cta.txt).
// NWAP_HOIST=0 keeps the per-row dispatch with one shared epilogue.
#ifndef NWAP_HOIST
#define NWAP_HOIST 1
#endif
// NWAP_HOIST_FASTONLY=1 (default; +1.0 % at 100k words, -0.9 % at 20k): the hoisted bodies serve only "fast" chunks (full chunk, every row valid over the
// whole window: no la == 0 test, no per-lane range checks, no slow emit in the body); everything else goes
// through the compact per-row-dispatch family with its one shared epilogue.
#ifndef NWAP_HOIST_FASTONLY
#define NWAP_HOIST_FASTONLY 1
#endif
#ifndef NWAP_ROW_PREFETCH
#define NWAP_ROW_PREFETCH 1
#endif
template <int LB, int FLAVOR, bool FASTONLY, class SM>
__device__ __forceinline__ void nwap_chunk_rows_h(SM &sm, const nwap_scheme_consts &sc, const uint32_t *nb,
                                                  const nwap_lane_cols &c, int mixmode, bool fast, int want_hist,
                                                  nwap_lane_stats &ls, nwap_chunk_acc &ca)
{
    const bool deep = mixmode > 2;
    if (FASTONLY && NWAP_ROW_PREFETCH) {
        // every row of a fast chunk is live: fetch the next row's {la, ala2, rowadj} (one LDS.128) a row ahead
        uint4 nxt = *reinterpret_cast<const uint4 *>(&sm.meta[0]);
#pragma unroll 1
        for (int rr = 0; rr < NWAP_R; ++rr) {
            const uint4 cur = nxt;
            nxt = *reinterpret_cast<const uint4 *>(&sm.meta[rr + 1 < NWAP_R ? rr + 1 : rr]);
            uint32_t v, vm1, vm2;
            nwap_row_dp<LB, FLAVOR>(sm.syms(rr, (int)cur.x), sm.ov, (int)cur.x, nb, c.l0, c.l1, sc, v, vm1, vm2, deep);
            if (mixmode == 1 || mixmode == 2) v = nwap_merge3(v, vm1, vm2, c);
            nwap_emit(sm, sm.meta[rr], cur.z, (int)cur.w, v, c, nwap_true(), 0, ls, ca);
        }
        return;
    }
#pragma unroll 1
    for (int rr = 0; rr < NWAP_R; ++rr) {
        const nwap_row_meta &m = sm.meta[rr];
        const int la = m.la;
        if (!FASTONLY && la == 0) continue;
        uint32_t v, vm1, vm2;
        nwap_row_dp<LB, FLAVOR>(sm.syms(rr, la), sm.ov, la, nb, c.l0, c.l1, sc, v, vm1, vm2, deep);
        if (mixmode == 1 || mixmode == 2) v = nwap_merge3(v, vm1, vm2, c);
        if (FASTONLY) nwap_emit(sm, m, m.ala2, m.rowadj, v, c, nwap_true(), 0, ls, ca);
        else nwap_emit(sm, m, m.ala2, m.rowadj, v, c, fast, want_hist, ls, ca);
    }
}

template <int FLAVOR, int QMAX, int QW, bool FASTONLY, class SM>
__device__ __forceinline__ void nwap_run_chunk_h(int LB, SM &sm, const nwap_scheme_consts &sc,
                                                 const uint32_t (&w0)[QW], const uint32_t (&w1)[QW],
                                                 const nwap_lane_cols &c, int mixmode, bool fast,
                                                 int want_hist, nwap_lane_stats &ls)
{
    uint32_t nb[QMAX];
    nwap_unpack_cols<FLAVOR, QMAX, QW>(w0, w1, nb);
    nwap_chunk_acc ca; ca.acc = 0; ca.acc_hi = 0; ca.rows_fast = 0;
#define NWAP_CASE(n)                                                                                       \
    case n:                                                                                                \
        if (n <= QMAX) nwap_chunk_rows_h<(n <= QMAX ? n : 1), FLAVOR, FASTONLY>(sm, sc, nb, c, mixmode, fast, want_hist, ls, ca); \
        break;
    switch (LB) { NWAP_CASES_1_32 default: break; }
#undef NWAP_CASE
    nwap_close_chunk(ls, ca);
}


// shared-window loads by 32-bit address: one induction variable serves both the load and the loop test (with
// generic pointers ptxas keeps two copies of it, one per use)
__device__ __forceinline__ uint2 nwap_lds64(uint32_t addr)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t nwap_lds32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 nwap_lds128(uint32_t addr)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// cnt += STEP; returns the carry-out (ptxas: one IADD3 with a predicate destination that the loop branch uses)
template <int STEP>
__device__ __forceinline__ bool nwap_bump_carry(uint32_t &cnt)
{
    uint32_t c;
    asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, 0, 0;" : "+r"(cnt), "=r"(c) : "n"(STEP));
    return c != 0;
}
__device__ __forceinline__ void nwap_sts8(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.u8 [%0], %1;" :: "r"(addr), "r"(v));
}


// ---- table-driven cell, second shape (FLAVOR 3, round 2): ONE shared-memory load per packed cell -----------------
// nwap_dp_row_tab packs two COLUMN words against one row word, so a packed cell needs two table entries of the same
// table row, E[a_i][b0_j] and E[a_i][b1_j]: two LDS.U8, and the shared-memory pipe is the bound (9.3 TCUPS).  Here the
// two halves of a register belong to two ROW words (rows 2p and 2p+1 of the band) against ONE column word per lane:
// the packed cell needs E[a_i][b_j] | E[a'_i][b_j] << 16, which is ONE 32-bit load from the row pair's PROFILE
//     W[p][i][b] = E[a_{2p,i}][b] | E[a_{2p+1,i}][b] << 16          (K words per matrix row, built per band)
// at the lane's column symbol -- the cell is LDS.32, subtract, add, VIMNMX3, as many instructions as the uniform
// scheme's.  The two row words differ in length: the pair runs min(la, la') matrix rows, captures the shorter word's
// final cell, runs on to max(la, la') and captures the other (one loop, entered twice).  The boundary column is the
// same for both halves (BIAS + i*u), so it is kept in a register and bumped per row.  The lane's two columns run as
// two independent chains in the same loop.  Profiles: 8 pairs x lmax rows x K words -- 30 KB at 40 symbols and 24 rows; the
// launch enables this shape when they fit (p.tab2_lmax > 0), and it serves the chunks the fast family serves (full,
// every row live, at most three lengths); everything else runs nwap_run_chunk_tab.
struct alignas(16) nwap_pair_meta {
    int lmin, lmax;            // matrix rows of the shorter / longer word of the pair
    uint32_t sel;              // halves of the SHORTER word: 0x0000ffff (row 2p) or 0xffff0000 (row 2p+1)
    uint32_t ala2;             // row potentials: alpha*la(2p) | alpha*la(2p+1) << 16
    int rowadj0, rowadj1;      // staged-byte bases of the two rows (nwap_row_meta::rowadj)
    int pad0, pad1;
};
#define NWAP_TAB2_PAIRS (NWAP_R / 2)
// Profile entries are 16 bits, E | E' << 8 (every E fits a byte): with 32-bit entries an alphabet of more than 32
// symbols puts two symbols on one shared-memory bank, and a warp's 32 column symbols then hit such a pair in nine
// loads out of ten (ncu at 40 symbols: 1.78 wavefronts per load, the shared-memory pipe 86 % busy -- THE bound of this
// cell).  Two 16-bit entries share a bank WORD, which is a broadcast, so alphabets of up to 64 symbols are
// conflict-free; the price is one byte permute per packed cell (E | E' << 8  ->  E | E' << 16).
#ifndef NWAP_TAB2_16
#define NWAP_TAB2_16 1
#endif
#if NWAP_TAB2_16
typedef uint16_t nwap_prof_t;
__device__ __forceinline__ uint32_t nwap_prof_load(const char *p) { return __byte_perm((uint32_t)*reinterpret_cast<const uint16_t *>(p), 0u, 0x4140u); }
#else
typedef uint32_t nwap_prof_t;
__device__ __forceinline__ uint32_t nwap_prof_load(const char *p) { return *reinterpret_cast<const uint32_t *>(p); }
#endif
// bytes of the profiles of one band, rounded up so that the pair records behind them stay 16-byte aligned
__host__ __device__ inline size_t nwap_tab2_prof_bytes(int lmax_rows, int K)
{
    return ((size_t)sizeof(nwap_prof_t) * NWAP_TAB2_PAIRS * (size_t)lmax_rows * (size_t)K + 15u) & ~size_t(15);
}

// Both of the lane's columns are scored in the same loop (two independent chains: the load -> subtract -> max3
// latency of one hides behind the other; these builds run one CTA per SM, so registers are plentiful).
template <int LB, int QW, class SM>
__device__ __forceinline__ void nwap_chunk_rows_tab2(SM &sm, const nwap_scheme_consts &sc, const uint32_t (&w0)[QW],
                                                     const uint32_t (&w1)[QW], const nwap_lane_cols &c, int K,
                                                     int lmax_rows, const nwap_prof_t *wprof, const nwap_pair_meta *pm,
                                                     nwap_lane_stats &ls)
{
    constexpr uint32_t ES = sizeof(nwap_prof_t);
    uint32_t ca[LB], cb[LB];                                     // column symbols as byte offsets in a profile row
#pragma unroll
    for (int j = 0; j < LB; ++j) { ca[j] = ES * nwap_byte_of(w0, j); cb[j] = ES * nwap_byte_of(w1, j); }
    const uint32_t kva = c.l0 == LB ? 0xffffffffu : 0u, k1a = c.l0 == LB - 1 ? 0xffffffffu : 0u;
    const uint32_t kvb = c.l1 == LB ? 0xffffffffu : 0u, k1b = c.l1 == LB - 1 ? 0xffffffffu : 0u;
    const uint32_t kposa = (uint32_t)(sc.beta * c.l0) * 65537u, kposb = (uint32_t)(sc.beta * c.l1) * 65537u;
    uint32_t acc = 0, acc_hi = 0;
    uint8_t *oa = sm.out + c.off0, *ob = sm.out + c.off1;
#pragma unroll 1
    for (int pr = 0; pr < NWAP_TAB2_PAIRS; ++pr) {
        const nwap_pair_meta m = pm[pr];
        const char *wr = reinterpret_cast<const char *>(wprof + (size_t)pr * lmax_rows * K);
        uint32_t Pa[LB + 1], Pb[LB + 1];
#pragma unroll
        for (int j = 0; j <= LB; ++j) { Pa[j] = NWAP_BIAS2; Pb[j] = NWAP_BIAS2; }
        uint32_t b0 = NWAP_BIAS2;                                // H'[i-1][0], the same for both halves and both columns
                                                                 // (H'[i][0] itself is dominated: nwap_dp_row, DOM)
        uint32_t va0 = 0, va1 = 0, vb0 = 0, vb1 = 0;
        int rows = m.lmin;
#pragma unroll 1
        for (int ph = 0; ph < 2; ++ph) {
#pragma unroll 1
            for (; rows > 0; --rows) {
                uint32_t lefta = 0, leftb = 0;
                uint32_t dwa = b0 - nwap_prof_load(wr + ca[0]);
                uint32_t dwb = b0 - nwap_prof_load(wr + cb[0]);
#pragma unroll
                for (int j = 1; j <= LB; ++j) {
                    uint32_t na = 0, nb_ = 0;
                    if (j < LB) {
                        na = Pa[j] - nwap_prof_load(wr + ca[j]);
                        nb_ = Pb[j] - nwap_prof_load(wr + cb[j]);
                    }
                    const uint32_t cura = j == 1 ? nwap_vmaxs2(dwa, Pa[j] + sc.u2) : nwap_vimax3_s16x2(dwa, Pa[j] + sc.u2, lefta);
                    const uint32_t curb = j == 1 ? nwap_vmaxs2(dwb, Pb[j] + sc.u2) : nwap_vimax3_s16x2(dwb, Pb[j] + sc.u2, leftb);
                    Pa[j] = cura; lefta = cura; dwa = na;
                    Pb[j] = curb; leftb = curb; dwb = nb_;
                }
                b0 += sc.u2;
                wr += ES * K;
            }
            const uint32_t ta = (Pa[LB >= 2 ? LB - 1 : LB] & k1a) | (Pa[LB >= 3 ? LB - 2 : LB] & ~k1a);
            const uint32_t tb = (Pb[LB >= 2 ? LB - 1 : LB] & k1b) | (Pb[LB >= 3 ? LB - 2 : LB] & ~k1b);
            const uint32_t fa = (Pa[LB] & kva) | (ta & ~kva), fb = (Pb[LB] & kvb) | (tb & ~kvb);
            if (ph == 0) { va0 = fa; vb0 = fb; } else { va1 = fa; vb1 = fb; }
            rows = m.lmax - m.lmin;
        }
        // halves: score + BIAS of (row 2p, column) and (row 2p+1, column)
        const uint32_t t_a = ((va0 & m.sel) | (va1 & ~m.sel)) + m.ala2 + kposa;
        const uint32_t t_b = ((vb0 & m.sel) | (vb1 & ~m.sel)) + m.ala2 + kposb;
        oa[m.rowadj0] = (uint8_t)t_a; oa[m.rowadj1] = (uint8_t)(t_a >> 16);
        ob[m.rowadj0] = (uint8_t)t_b; ob[m.rowadj1] = (uint8_t)(t_b >> 16);
        ls.mn2 = __vmins2(__vmins2(ls.mn2, t_a), t_b);
        ls.mx2 = __vmaxs2(__vmaxs2(ls.mx2, t_a), t_b);
        acc += t_a; acc_hi += t_a >> 16;
        acc += t_b; acc_hi += t_b >> 16;
    }
    ls.sum += (long long)(acc - (acc_hi << 16)) + (long long)acc_hi - 4ll * NWAP_TAB2_PAIRS * (long long)NWAP_BIAS;
    ls.count += 4 * NWAP_TAB2_PAIRS;
}

template <int QMAX, int QW, class SM>
__device__ __forceinline__ void nwap_run_chunk_tab2(int LB, SM &sm, const nwap_scheme_consts &sc,
                                                    const uint32_t (&w0)[QW], const uint32_t (&w1)[QW],
                                                    const nwap_lane_cols &c, int K, int lmax_rows, const nwap_prof_t *wprof,
                                                    const nwap_pair_meta *pm, nwap_lane_stats &ls)
{
#define NWAP_CASE(n)                                                                                       \
    case n:                                                                                                \
        if (n <= QMAX) nwap_chunk_rows_tab2<(n <= QMAX ? n : 1), QW>(sm, sc, w0, w1, c, K, lmax_rows, wprof, pm, ls); \
        break;
    switch (LB) { NWAP_CASES_1_32 default: break; }
#undef NWAP_CASE
}


// ---- the fast family, second shape (NWAP_FAST2=1) -------------------------------------------------------------
// Serves chunks that are full, whose rows all cover the whole column window, and whose lanes span at most three
// word lengths (mixmode <= 2) -- everything else goes through the compact per-row-dispatch family.  Compared with
// nwap_chunk_rows_h it executes fewer instructions per row word:
//   * no deep select and no mixmode tests: the final cell is always merged from the last three columns;
//   * the column codes are unpacked inside the length body (LB of them, not QMAX: three PRMT per two columns);
//   * shared memory is addressed through 32-bit shared-window addresses, rows and metadata walked by pointer
//     (meta[] has one readable record past the band: the next row's record is fetched a row ahead);
//   * the matrix-row loop is counted by carry and carries no border column: three control instructions per matrix
//     row (LDS.64, IADD3, branch);
//   * bodies up to NWAP_F2_DUFF_MAXLB run two matrix rows per loop trip (four control instructions per two rows;
//     beyond LB 8 the doubled body loses to instruction-cache misses).
// A peeled first matrix row (three instructions per cell, no initialisation of the rolling row) executes 2 * LB
// fewer instructions per row word and is still SLOWER (-1.8 % for LB <= 8 ... -3.7 % for all bodies): code size.
// A/B records: profiles/r02a_ab_fast2.txt, profiles/r02c_ab_rowloop.txt.
#ifndef NWAP_FAST2
#define NWAP_FAST2 1
#endif
#ifndef NWAP_F2_DUFF_MAXLB
#define NWAP_F2_DUFF_MAXLB 8
#endif
template <int LB, int FLAVOR, int QW, class SM>
__device__ __forceinline__ void nwap_chunk_rows_fast2(SM &sm, const nwap_scheme_consts &sc, const uint32_t (&w0)[QW],
                                                      const uint32_t (&w1)[QW], const nwap_lane_cols &c,
                                                      nwap_lane_stats &ls)
{
    uint32_t nb[LB];
    nwap_unpack_cols<FLAVOR, LB, QW>(w0, w1, nb);
    uint32_t acc = 0, acc_hi = 0;
    const uint32_t out_s = (uint32_t)__cvta_generic_to_shared(sm.out);
    const uint32_t o0 = out_s + c.off0, o1 = out_s + c.off1;
    // through a shuffle: opaque to ptxas, which otherwise re-derives beta * lengths with a constant load per row word
    const uint32_t kpos2 = __shfl_sync(0xffffffffu, c.kpos2, (int)(threadIdx.x & 31u));
    static_assert(SM::END_ALIGNED, "fast2 serves the uniform-scheme builds");
    uint32_t sym_s = (uint32_t)__cvta_generic_to_shared(sm.syms(0, 0));       // END of row 0's records
    uint32_t meta_s = (uint32_t)__cvta_generic_to_shared(&sm.meta[0]);
    constexpr uint32_t SYM_PITCH = sizeof(sm.rowsym[0]);
    constexpr uint32_t META_PITCH = sizeof(nwap_row_meta);
    uint4 nxt = nwap_lds128(meta_s);
#pragma unroll 1
    for (int rr = 0; rr < NWAP_R; ++rr) {
        // the whole 16-byte record {la, -8 * la, ala2, rowadj} is fetched a row ahead
        const uint32_t nxt_cnt = nxt.y;
        const uint2 cur = make_uint2(nxt.z, nxt.w);
        meta_s += META_PITCH;
        nxt = nwap_lds128(meta_s);                               // meta[] has one readable record past the band
        uint32_t P[LB + 1];
        const uint32_t sa = sym_s;
        sym_s += SYM_PITCH;
        // The row's records END at sa (warp-uniform: a uniform register); the counter -8 * la runs up to zero and the
        // carry-out of its increment IS the loop test: LDS.64 [cnt + base], IADD3 (carry), branch -- three control
        // instructions per matrix row (pointer bump + compare + move + branch + load were five).  The border column
        // needs no register: see nwap_dp_row<.., DOM>.
#pragma unroll
        for (int j = 1; j <= LB; ++j) P[j] = NWAP_BIAS2;         // H'[0][j]
        uint32_t cnt = nxt_cnt;
        bool done;
        if (LB <= NWAP_F2_DUFF_MAXLB) {
            // two matrix rows per loop trip; a word of odd length enters at the second copy
            if (cnt & 8u) { cnt -= 8u; goto second_row; }
#pragma unroll 1
            do {
                {
                    const uint2 x = nwap_lds64(sa + cnt);
                    nwap_dp_row<LB, FLAVOR, true>(x.x, nb, P, x.y, 0u, sc);
                }
            second_row:
                {
                    const uint2 x = nwap_lds64(sa + cnt + 8u);
                    done = nwap_bump_carry<16>(cnt);
                    nwap_dp_row<LB, FLAVOR, true>(x.x, nb, P, x.y, 0u, sc);
                }
            } while (!done);
        } else {
#pragma unroll 1
            do {                                                 // la >= 1 always
                const uint2 x = nwap_lds64(sa + cnt);
                done = nwap_bump_carry<8>(cnt);
                nwap_dp_row<LB, FLAVOR, true>(x.x, nb, P, x.y, 0u, sc);
            } while (!done);
        }
        const uint32_t v = nwap_merge3(P[LB], P[LB >= 2 ? LB - 1 : LB], P[LB >= 3 ? LB - 2 : LB], c);
        const uint32_t t = v + cur.x + kpos2;                    // halves: score + BIAS
        const uint32_t thi = t >> 16;
        nwap_sts8(o0 + cur.y, t);
        nwap_sts8(o1 + cur.y, thi);
        ls.mn2 = __vmins2(ls.mn2, t);
        ls.mx2 = __vmaxs2(ls.mx2, t);
        acc += t; acc_hi += thi;                                 // packed sums, separated once per chunk
    }
    ls.sum += (long long)(acc - (acc_hi << 16)) + (long long)acc_hi - 2ll * NWAP_R * (long long)NWAP_BIAS;
    ls.count += 2 * NWAP_R;
}

template <int FLAVOR, int QMAX, int QW, class SM>
__device__ __forceinline__ void nwap_run_chunk_fast2(int LB, SM &sm, const nwap_scheme_consts &sc,
                                                     const uint32_t (&w0)[QW], const uint32_t (&w1)[QW],
                                                     const nwap_lane_cols &c, nwap_lane_stats &ls)
{
#define NWAP_CASE(n)                                                                                       \
    case n:                                                                                                \
        if (n <= QMAX) nwap_chunk_rows_fast2<(n <= QMAX ? n : 1), FLAVOR, QW>(sm, sc, w0, w1, c, ls);      \
        break;
    switch (LB) { NWAP_CASES_1_32 default: break; }
#undef NWAP_CASE
}


// Tried and rejected this round (same-box A/B, evidence in profiles/r01c..r01e and git history):
// hoisting the length dispatch out of the row loop, one symbol stream per band, dual-chain
// chunks (4 columns per lane), a cold code family for chunks spanning >= 3 lengths.

__device__ __forceinline__ void nwap_stage_sym(nwap_sym2 &x, uint32_t a, const nwap_scheme_consts &sc, uint32_t d0, const nwap_ov_part *, int)
{
    x.a2 = nwap_row_code(a, sc); x.d0 = d0;
}
__device__ __forceinline__ void nwap_stage_sym(nwap_sym8 &, uint32_t, const nwap_scheme_consts &, uint32_t, const nwap_ov_part *, int)
{
    // override schemes stage whole rows (nwap_stage_row_ov, one thread per row: the row potential is a prefix sum)
}

// One chunk whose longest word exceeds the register-resident row: block-wise DP (nwap_dp_blocks), per-lane
// selection of the final cell, shared epilogue.  Rare by construction (words of 25..64 symbols in a wide
// build).  Inlined: out of line (generic addressing of the shared row symbols, call ABI) the wide build lost
// 3.1 % on a vocabulary with no long word at all, inlined 1.4 % (gpurun A/B, 100,000 words).
#ifndef NWAP_WIDE_INLINE
#define NWAP_WIDE_INLINE 1
#endif
#if NWAP_WIDE_INLINE
#define NWAP_WIDE_ATTR __forceinline__
#else
#define NWAP_WIDE_ATTR __noinline__
#endif
template <int FLAVOR, class SM>
__device__ NWAP_WIDE_ATTR void nwap_run_chunk_wide(int LB, SM &sm, const nwap_scheme_consts &sc, const uint8_t *b0,
                                                 const uint8_t *b1, const nwap_lane_cols &c, bool fast, int want_hist,
                                                 nwap_lane_stats &ls)
{
    nwap_chunk_acc ca; ca.acc = 0; ca.acc_hi = 0; ca.rows_fast = 0;
    const int nblk = (LB + NWAP_WB - 1) / NWAP_WB;
    uint32_t save[NWAP_MAXLEN_WIDE + 1];
#pragma unroll 1
    for (int rr = 0; rr < NWAP_R; ++rr) {
        const nwap_row_meta &m = sm.meta[rr];
        const int la = m.la;
        if (la == 0) continue;
        const nwap_sym2 *rs = reinterpret_cast<const nwap_sym2 *>(sm.syms(rr, la));
        const uint32_t v = FLAVOR == 3 ? nwap_dp_blocks_tab(rs, la, b0, b1, nblk, c.l0, c.l1, sc, save, sm.etab)
                                       : nwap_dp_blocks(rs, la, b0, b1, nblk, c.l0, c.l1, sc, save);
        nwap_emit(sm, m, m.ala2, m.rowadj, v, c, fast, want_hist, ls, ca);
    }
    nwap_close_chunk(ls, ca);
}

// Sparse-output scan of one staged row segment (one warp): 16 staged scores per lane per trip, SWAR compare,
// and -- rarely -- a warp-aggregated append of (index, score) keys plus the two degree increments.
struct nwap_sparse_consts {
    uint32_t lo_rep, hi_rep;
    bool lo_th, hi_th, all_lo, has_hi;
};
__device__ __forceinline__ nwap_sparse_consts nwap_make_sparse_consts(const nwap_sparse_out &so)
{
    nwap_sparse_consts k;
    const int lo = so.mode == 1 ? so.threshold : so.gmin;          // candidates: score >= lo ...
    const int hi = so.mode == 1 ? 127 : so.gmax;                   // ... and score <= hi
    const uint32_t Tlo = (uint32_t)(max(lo, -128) + 128);
    k.lo_rep = (Tlo & 0x7fu) * 0x01010101u; k.lo_th = (Tlo & 0x80u) != 0; k.all_lo = lo <= -128;
    const uint32_t Thi = (uint32_t)(min(hi, 126) + 1 + 128);
    k.hi_rep = (Thi & 0x7fu) * 0x01010101u; k.hi_th = (Thi & 0x80u) != 0; k.has_hi = hi < 127;
    return k;
}

template <class SM>
__device__ __forceinline__ void nwap_sparse_row(SM &sm, const nwap_tile_params &p, const nwap_sparse_consts &k,
                                                int rr, int64_t row, int64_t strip_lo, int lane)
{
    const nwap_row_meta &m = sm.meta[rr];
    const int seg = m.seglen;
    if (seg <= 0) return;
    const nwap_sparse_out &so = p.sparse;
    if (so.mode == 1 ? so.threshold > 127 : so.gmin > so.gmax) return;       // nothing can be kept
    const int skew = nwap_meta_skew<SM::PITCH>(m, rr);
    const uint8_t *rowbase = sm.out + rr * SM::PITCH;           // 16-byte aligned; the segment starts at +skew
    const int nvec = (skew + seg + 15) >> 4;
    for (int v0 = 0; v0 < nvec; v0 += 32) {
        const int v = v0 + lane;
        unsigned bits = 0;
        if (v < nvec) {
            const uint4 x = *reinterpret_cast<const uint4 *>(rowbase + 16 * v);
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                unsigned ok = k.all_lo ? 0xfu : nwap_ge_bits4(w[q], k.lo_rep, k.lo_th);
                if (k.has_hi) ok &= ~nwap_ge_bits4(w[q], k.hi_rep, k.hi_th);
                bits |= ok << (4 * q);
            }
            const int first = skew - 16 * v;                     // vector bytes before the segment
            if (first > 0) bits &= 0xffffu << first;
            const int last = skew + seg - 16 * v;                // vector bytes up to the segment's end
            if (last < 16) bits &= (1u << last) - 1u;
        }
        if (!__any_sync(0xffffffffu, bits != 0u)) continue;
        if (so.mode == 2 && bits) {                              // per-length bounds of the reference's float64 test
            unsigned keep = 0, rest = bits;
            while (rest) {
                const int j = __ffs(rest) - 1;
                rest &= rest - 1;
                const int sc8 = (int)(int8_t)rowbase[16 * v + j];
                const int lc = (int)p.lens[strip_lo + m.clo_off + (16 * v + j - skew)];
                const short2 bnd = sm.kbounds[max(m.la, lc)];
                if (sc8 >= (int)bnd.x && sc8 <= (int)bnd.y) keep |= 1u << j;
            }
            bits = keep;
        }
        const int cnt = __popc(bits);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(so.count, (unsigned long long)total);
        base = __shfl_sync(0xffffffffu, base, 31);
        long long pos = (long long)base + (incl - cnt);
        while (bits) {
            const int j = __ffs(bits) - 1;
            bits &= bits - 1;
            const int b = 16 * v + j - skew;                     // offset inside the segment
            const unsigned long long idx = (unsigned long long)(p.start + m.g0 + b);
            if (pos < so.cap) so.keys[pos] = (idx << 8) | (unsigned long long)rowbase[16 * v + j];
            if (so.degree) {
                atomicAdd(&so.degree[row], 1);
                atomicAdd(&so.degree[strip_lo + m.clo_off + b], 1);
            }
            ++pos;
        }
    }
}

// QMAX = register-resident row width (16, 24 or 32): the longest word the instantiation
// accepts.  Stored word rows are qpad = 16 or 32 bytes; QW 32-bit words of them are loaded.
// WIDE: words of up to NWAP_MAXLEN_WIDE = 64 symbols are accepted; chunks whose longest word exceeds QMAX take the
// block-wise path (nwap_run_chunk_wide), everything else runs the same length-specialised bodies.
// CMP: sparse-output mode (p.sparse): the flush stage scans the staged scores for kept edges; the dense store
// happens only when p.out is non-NULL.
template <int FLAVOR, int QMAX, bool OV, bool WIDE = false, bool CMP = false>
__global__ void __launch_bounds__(NWAP_THREADS, ((OV || FLAVOR == 3) ? 1 : NWAP_MINB))   // sparse-override builds run one CTA per SM (two lose: profiles/r02b_overrides.txt); so do the table builds (their row-pair profiles fill the shared memory)
k_score_tiles(const nwap_tile_params p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int MAXL = WIDE ? NWAP_MAXLEN_WIDE : QMAX;          // longest word accepted
    typedef nwap_tile_smem_t<(OV ? 1 : (FLAVOR == 3 ? 2 : 0)), (WIDE ? NWAP_MAXLEN_WIDE : NWAP_MAXLEN_FAST)> smem_t;
    constexpr int SYMLEN = WIDE ? NWAP_MAXLEN_WIDE : NWAP_MAXLEN_FAST;   // row symbols staged per row
    smem_t &sm = *reinterpret_cast<smem_t *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const nwap_scheme_consts sc = p.sc;
    constexpr int QW = QMAX <= 16 ? 4 : 8;
    static_assert(!WIDE || ((FLAVOR == 1 || FLAVOR == 3) && !OV && QMAX == 24), "the wide build exists for the default uniform-scheme cell and the table-driven cell");

    if (tid == 0) { sm.sum = 0; sm.count = 0; sm.mn = 127; sm.mx = -128; }
    // the 256-bin histogram is not accumulated here: a request for it is served by k_payload_stats over the
    // scored bytes (5.5 TB/s), so every chunk keeps the fast emit (per-edge shared atomics cost far more)
    constexpr int kNoHist = 0;
    if (FLAVOR == 3) {
        for (int w = tid; w < p.ov_K * p.ov_K; w += NWAP_THREADS) sm.etab[w] = p.etab[w];
    }
    // FLAVOR 3, second shape: row-pair profiles and pair records behind the table (dynamic shared memory, sized by the launch)
    nwap_prof_t *const tab2_prof = reinterpret_cast<nwap_prof_t *>(sm.etab + (((size_t)p.ov_K * p.ov_K + 15u) & ~size_t(15)));
    nwap_pair_meta *const tab2_pm = reinterpret_cast<nwap_pair_meta *>(reinterpret_cast<char *>(tab2_prof) + nwap_tab2_prof_bytes(p.tab2_lmax, p.ov_K));
    if (CMP && p.sparse.mode == 2)
        for (int b = tid; b < 256; b += NWAP_THREADS) sm.kbounds[b] = p.sparse.bounds[b];
    const nwap_sparse_consts skc = nwap_make_sparse_consts(p.sparse);
    if (OV) {
        for (int k = tid; k < p.ov_K; k += NWAP_THREADS) {
            const nwap_ov_row t = p.ov_table[k];
            nwap_ov_part y;
            y.p0 = t.b2[0]; y.nd0 = t.nd[0]; y.p1 = t.b2[1]; y.nd1 = t.nd[1];
            sm.ov[k] = y;
        }
    }
    nwap_lane_stats ls;
    ls.mn2 = 0x7fff7fffu; ls.mx2 = 0u; ls.sum = 0; ls.count = 0;

    for (;;) {
        __syncthreads();
        if (tid == 0) sm.unit = atomicAdd(p.unit_counter, 1ULL);
        __syncthreads();
        const int64_t t = (int64_t)sm.unit;
        if (t >= p.unit_count) break;

        int64_t group, strip;
        nwap_unit_decode(p.us, p.unit_begin + t, &group, &strip);
        constexpr int CW = smem_t::C;                    // strip width of this build (p.us was laid out for it)
        const int64_t strip_lo = strip * CW;
        const int64_t strip_hi = min(strip_lo + (int64_t)CW, p.n);
        const int64_t grow0 = group * (int64_t)p.us.gb * NWAP_R;
        const int64_t rmin = max(grow0, p.r_first);
        const int64_t rmax = min(grow0 + (int64_t)p.us.gb * NWAP_R - 1, p.r_last);
        if (rmin > rmax) continue;
        const int64_t cwin_lo = max(strip_lo, rmin + 1);
        if (cwin_lo >= strip_hi) continue;

        // ---- counting sort of the unit's columns by word length, longest first ----
        for (int b = tid; b < NWAP_WARPS * (SYMLEN + 2); b += NWAP_THREADS) (&sm.bins[0][0])[b] = 0;
        __syncthreads();
        constexpr int PER = CW / NWAP_THREADS;         // 16 columns per thread (8 with half-width strips)
        static_assert(PER == 16 || PER == 8, "one aligned uint4 / uint2 of lengths per thread");
        uint32_t lw[PER / 4];
        if constexpr (PER == 16) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p.lens + strip_lo) + tid);
            lw[0] = v.x; lw[1] = v.y; lw[2] = v.z; lw[3] = v.w;
        } else {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p.lens + strip_lo) + tid);
            lw[0] = v.x; lw[1] = v.y;
        }
        const int kbase = tid * PER;
        const int win_lo = (int)(cwin_lo - strip_lo), win_hi = (int)(strip_hi - strip_lo);
        // In the strip that holds the unit's own rows (the diagonal strip) the columns up to the unit's last row are
        // valid for some of its rows only.  They are sorted BEHIND all the others (bin 0), so that every chunk of the
        // clean part [0, nclean) is valid for every row of every band of the unit and takes the fast path; the few
        // chunks behind it (at most gb * 16 columns) take the path with per-lane range checks.
        const int dirty_hi = (int)max((int64_t)0, min((int64_t)CW, grow0 + (int64_t)p.us.gb * NWAP_R - strip_lo));
        // zero the lengths of columns outside the window (and clamp, defensively)
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int k = kbase + e;
            uint32_t len = nwap_byte_of(lw, e);
            if (k < win_lo || k >= win_hi) len = 0;
            if (len > (uint32_t)MAXL) len = MAXL;
            lw[e >> 2] = (lw[e >> 2] & ~(0xffu << (8 * (e & 3)))) | (len << (8 * (e & 3)));
        }
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int len = (int)nwap_byte_of(lw, e);
            if (len) atomicAdd(&sm.bins[warp][kbase + e < dirty_hi ? 0 : len], 1);
        }
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int len = MAXL; len >= 1; --len)
                for (int w = 0; w < NWAP_WARPS; ++w) { int cnt = sm.bins[w][len]; sm.bins[w][len] = run; run += cnt; }
            sm.nclean = run;
            for (int w = 0; w < NWAP_WARPS; ++w) { int cnt = sm.bins[w][0]; sm.bins[w][0] = run; run += cnt; }
            sm.ncols = run;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int len = (int)nwap_byte_of(lw, e);
            if (len) {
                const int pos = atomicAdd(&sm.bins[warp][kbase + e < dirty_hi ? 0 : len], 1);
                sm.cols[pos] = (uint16_t)(kbase + e);
                sm.clen[pos] = (uint8_t)len;
            }
        }

        // ---- bands of the group ----
        for (int b = 0; b < p.us.gb; ++b) {
            const int64_t rb0 = grow0 + (int64_t)b * NWAP_R;
            if (rb0 + NWAP_R - 1 < rmin || rb0 > rmax) continue;
            __syncthreads();                         // previous flush done; sort scatter visible
            // stage row metadata
            if (tid < NWAP_R) {
                const int64_t r = rb0 + tid;
                nwap_row_meta m;
                m.la = 0; m.clo_off = 0; m.seglen = 0; m.rowadj = 0; m.ala2 = 0; m.symend = 0; m.g0 = 0;
                if (r >= rmin && r <= rmax) {
                    int64_t clo = max(strip_lo, r + 1);
                    int64_t chi = strip_hi;
                    if (r == p.r_first) clo = max(clo, p.c_start);
                    if (r == p.r_last) chi = min(chi, p.c_end + 1);
                    if (chi > clo) {
                        m.la = (int)p.lens[r];
                        m.clo_off = (int)(clo - strip_lo);
                        m.seglen = (int)(chi - clo);
                        m.g0 = nwap_before_row(r, p.n) + (clo - r - 1) - p.start;
                        const int skew = (int)((reinterpret_cast<uintptr_t>(p.out) + (uintptr_t)m.g0) & 15u);
                        m.rowadj = tid * smem_t::PITCH + skew - m.clo_off;
                        m.symend = (uint32_t)(-8 * m.la);
                        m.ala2 = (uint32_t)(sc.alpha * m.la * 65537);
                        if (OV) {
                            const int gsum = nwap_stage_row_ov(p.ids + r * p.qpad, m.la, p.ov_table, p.ov_K, sc,
                                                               reinterpret_cast<nwap_sym8 *>(&sm.rowsym[tid][0]));
                            m.ala2 = (uint32_t)((sc.alpha * m.la + gsum) * 65537);
                        }
                    }
                }
                sm.meta[tid] = m;
            }
            // stage row symbols, packed a*65537, with the row boundary values (4 symbols per item)
            for (int item = tid; !OV && item < NWAP_R * (SYMLEN / 4); item += NWAP_THREADS) {
                const int rr = item / (SYMLEN / 4), q4 = item % (SYMLEN / 4);
                const int64_t r = rb0 + rr;
                if (q4 < (WIDE ? (p.qpad >> 2) : QW) && r >= rmin && r <= rmax) {
                    const uint32_t v = __ldg(reinterpret_cast<const uint32_t *>(p.ids + r * p.qpad) + q4);
                    const int la_r = (int)p.lens[r];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t a = (v >> (8 * e)) & 0xffu;
                        if (q4 * 4 + e < la_r)           // slot [la] belongs to the boundary record
                            nwap_stage_sym(sm.syms(rr, la_r)[q4 * 4 + e], a, sc, NWAP_BIAS2 + (uint32_t)(q4 * 4 + e) * sc.u2,
                                           sm.ov, p.ov_K);
                    }
                }
            }
            // simple band: all R rows present and neither end of the launch range clips one of them; every row then
            // covers the whole CLEAN part of the sorted columns (columns beyond the unit's last row: in a strip to the
            // right of the unit's rows that is every column).  Evaluated by every thread from launch scalars: no
            // extra barrier, nothing read back from shared memory.
            const bool clip_first = p.r_first >= rb0 && p.r_first < rb0 + NWAP_R && p.c_start > strip_lo;
            const bool clip_last = p.r_last >= rb0 && p.r_last < rb0 + NWAP_R && p.c_end + 1 < strip_hi;
            const bool band_simple = rb0 >= rmin && rb0 + NWAP_R - 1 <= rmax && !clip_first && !clip_last;
            // FLAVOR 3, second shape: the band's rows are PAIRED BY LENGTH (a pair runs max(la, la') matrix rows for both
            // of its words: neighbours in the vocabulary waste 19 % of them at the French length distribution, neighbours
            // in length order 3 %).  Every warp ranks the 16 lengths for itself (lanes 0..15, shuffles only): t2row =
            // the band row whose length has rank `lane`, longest first, ties by row.
            const bool tab2_band = FLAVOR == 3 && p.tab2_lmax > 0 && band_simple;
            if (tab2_band) {
                // sm.t2order[k] = the band row whose length has rank k (longest first, ties by row)
                if (tid < NWAP_R) {
                    const uint8_t *bl = p.lens + rb0;
                    const int mylen = (int)bl[tid];
                    int rank = 0;
#pragma unroll
                    for (int j = 0; j < NWAP_R; ++j) {
                        const int lj = (int)bl[j];
                        rank += (lj > mylen || (lj == mylen && j < tid)) ? 1 : 0;
                    }
                    sm.t2order[rank] = (uint8_t)tid;
                }
                __syncthreads();
                // row-pair profiles of the band (nwap_chunk_rows_tab2): one (pair, matrix row) per thread
                const int lmx = p.tab2_lmax, K = p.ov_K;
                for (int item = tid; item < NWAP_TAB2_PAIRS * lmx; item += NWAP_THREADS) {
                    const int pr = item / lmx, i = item - pr * lmx;
                    const int64_t r0 = rb0 + sm.t2order[2 * pr], r1 = rb0 + sm.t2order[2 * pr + 1];
                    const int la0 = (int)p.lens[r0], la1 = (int)p.lens[r1];
                    if (i >= max(la0, la1)) continue;
                    const uint32_t a0 = i < la0 ? (uint32_t)p.ids[r0 * p.qpad + i] : 0u;
                    const uint32_t a1 = i < la1 ? (uint32_t)p.ids[r1 * p.qpad + i] : 0u;
                    const uint8_t *e0 = sm.etab + a0 * K, *e1 = sm.etab + a1 * K;
                    nwap_prof_t *w = tab2_prof + (size_t)item * K;
                    for (int b = 0; b < K; ++b) w[b] = (nwap_prof_t)((uint32_t)e0[b] | ((uint32_t)e1[b] << (4 * sizeof(nwap_prof_t))));
                }
            }
            if (tid == 0) sm.next_chunk = 0;
            __syncthreads();
            if (tab2_band) {
                if (tid < NWAP_TAB2_PAIRS) {
                    const nwap_row_meta &m0 = sm.meta[sm.t2order[2 * tid]], &m1 = sm.meta[sm.t2order[2 * tid + 1]];
                    nwap_pair_meta pm;
                    pm.lmin = min(m0.la, m1.la); pm.lmax = max(m0.la, m1.la);
                    pm.sel = m0.la <= m1.la ? 0x0000ffffu : 0xffff0000u;
                    pm.ala2 = (uint32_t)(sc.alpha * m0.la) + ((uint32_t)(sc.alpha * m1.la) << 16);
                    pm.rowadj0 = m0.rowadj; pm.rowadj1 = m1.rowadj; pm.pad0 = pm.pad1 = 0;
                    tab2_pm[tid] = pm;
                }
                __syncthreads();
            }

            // ---- compute: warps pull chunks of 64 sorted columns, longest first ----
            const int ncols = sm.ncols, nclean = sm.nclean;
            for (;;) {
                int item = 0;
                if (lane == 0) item = atomicAdd(&sm.next_chunk, 1);
                item = __shfl_sync(0xffffffffu, item, 0);
                const int kc = item * NWAP_CHUNK;
                if (kc >= ncols) break;
                // register width of the chunk: its longest word, optionally rounded up to a multiple of
                // NWAP_LBSTEP (fewer distinct length bodies in flight; the 3-level merge covers the slack)
                const int ka = kc + 2 * lane, kb = ka + 1;
                const bool va = ka < ncols, vb = kb < ncols;
                int la_ = va ? (int)sm.clen[ka] : 0, lb_ = vb ? (int)sm.clen[kb] : 0;
                const bool clean = kc + NWAP_CHUNK <= nclean;             // sorted part: the chunk's first word is its longest
                const int lraw = clean ? (int)sm.clen[kc] : __reduce_max_sync(0xffffffffu, max(la_, lb_));
                const int LB = min((lraw + NWAP_LBSTEP - 1) / NWAP_LBSTEP * NWAP_LBSTEP, MAXL);
                if (!va) la_ = LB;
                if (!vb) lb_ = LB;
                const uint32_t off0 = va ? (uint32_t)sm.cols[ka] : 0xffffu;
                const uint32_t off1 = vb ? (uint32_t)sm.cols[kb] : 0xffffu;
                // column words (invalid lanes re-read the chunk's first column; their results are dropped)
                const int64_t ca = strip_lo + (va ? sm.cols[ka] : sm.cols[kc]);
                const int64_t cb = strip_lo + (vb ? sm.cols[kb] : sm.cols[kc]);
                uint32_t w0[QW], w1[QW];
#pragma unroll
                for (int v = 0; v < QW / 4; ++v) {
                    const uint4 x = __ldg(reinterpret_cast<const uint4 *>(p.ids + ca * p.qpad) + v);
                    const uint4 y = __ldg(reinterpret_cast<const uint4 *>(p.ids + cb * p.qpad) + v);
                    w0[4 * v] = x.x; w0[4 * v + 1] = x.y; w0[4 * v + 2] = x.z; w0[4 * v + 3] = x.w;
                    w1[4 * v] = y.x; w1[4 * v + 1] = y.y; w1[4 * v + 2] = y.z; w1[4 * v + 3] = y.w;
                }
                const nwap_lane_cols cA = nwap_make_lane_cols(off0, off1, la_, lb_, LB, sc);
                const int lmin = __reduce_min_sync(0xffffffffu, min(la_, lb_));
                const int mixmode = min(LB - lmin, 3);      // 0: uniform, 1/2: last two/three columns, 3: deep
                const bool fast = band_simple && clean;
                if (WIDE && LB > QMAX) {
                    nwap_run_chunk_wide<FLAVOR>(LB, sm, sc, p.ids + ca * p.qpad, p.ids + cb * p.qpad, cA, fast, kNoHist, ls);
                    continue;
                }
                if (FLAVOR == 3) {
                    if (p.tab2_lmax > 0 && fast && mixmode <= 2)
                        nwap_run_chunk_tab2<QMAX, QW>(LB, sm, sc, w0, w1, cA, p.ov_K, p.tab2_lmax, tab2_prof, tab2_pm, ls);
                    else
                        nwap_run_chunk_tab<QMAX, QW>(LB, sm, sc, w0, w1, cA, mixmode, fast, kNoHist, ls);
                    continue;
                }
#if NWAP_HOIST
                // two code families only where the register budget allows (the 32-wide and sparse-override
                // instantiations would spill): there the hoisted bodies also carry the slow emit
                constexpr bool FASTONLY = NWAP_HOIST_FASTONLY && QMAX <= 24 && !OV;
#if NWAP_FAST2
                if constexpr (FASTONLY && FLAVOR == 1) {
                    if (fast && mixmode <= 2) nwap_run_chunk_fast2<FLAVOR, QMAX, QW>(LB, sm, sc, w0, w1, cA, ls);
                    else nwap_run_chunk<FLAVOR, QMAX, QW>(LB, sm, sc, w0, w1, cA, mixmode, fast, kNoHist, ls);
                    continue;
                }
#endif
                if (!FASTONLY || fast) nwap_run_chunk_h<FLAVOR, QMAX, QW, FASTONLY>(LB, sm, sc, w0, w1, cA, mixmode, fast, kNoHist, ls);
                else nwap_run_chunk<FLAVOR, QMAX, QW>(LB, sm, sc, w0, w1, cA, mixmode, fast, kNoHist, ls);
#else
                nwap_run_chunk<FLAVOR, QMAX, QW>(LB, sm, sc, w0, w1, cA, mixmode, fast, kNoHist, ls);
#endif
            }
            __syncthreads();

            // ---- sparse output: scan the staged rows for kept edges ----
            if (CMP) {
                for (int rr = warp; rr < NWAP_R; rr += NWAP_WARPS) nwap_sparse_row(sm, p, skc, rr, rb0 + rr, strip_lo, lane);
                if (p.out == nullptr) continue;          // no dense payload wanted (uniform across the grid)
            }
            // ---- flush: each warp copies whole row segments, 16 B aligned in both spaces ----
            for (int rr = warp; rr < NWAP_R; rr += NWAP_WARPS) {
                const int seg = sm.meta[rr].seglen;
                if (seg <= 0) continue;
                const int skew = nwap_meta_skew<smem_t::PITCH>(sm.meta[rr], rr);
                const uint8_t *src = sm.out + rr * smem_t::PITCH + skew;
                int8_t *dst = p.out + sm.meta[rr].g0;
                int head = (16 - skew) & 15;
                if (head > seg) head = seg;
                if (lane < head) dst[lane] = (int8_t)src[lane];
                const int nvec = (seg - head) >> 4;
                const uint4 *s4 = reinterpret_cast<const uint4 *>(src + head);
                uint4 *d4 = reinterpret_cast<uint4 *>(dst + head);
                for (int v = lane; v < nvec; v += 32) d4[v] = s4[v];
                const int tail0 = head + (nvec << 4);
                if (tail0 + lane < seg) dst[tail0 + lane] = (int8_t)src[tail0 + lane];
            }
        }
    }

    // ---- statistics: thread -> warp -> CTA -> global ----
    long long wsum = ls.sum, wcnt = ls.count;
    int tmn = min((int)(ls.mn2 & 0xffffu), (int)(ls.mn2 >> 16)) - (int)NWAP_BIAS;
    int tmx = max((int)(ls.mx2 & 0xffffu), (int)(ls.mx2 >> 16)) - (int)NWAP_BIAS;
    if (ls.count == 0) { tmn = 127; tmx = -128; }
    tmn = min(tmn, 127); tmx = max(tmx, -128);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
        wcnt += __shfl_xor_sync(0xffffffffu, wcnt, o);
        tmn = min(tmn, __shfl_xor_sync(0xffffffffu, tmn, o));
        tmx = max(tmx, __shfl_xor_sync(0xffffffffu, tmx, o));
    }
    __syncthreads();
    if (lane == 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&sm.sum), (unsigned long long)wsum);
        atomicAdd(reinterpret_cast<unsigned long long *>(&sm.count), (unsigned long long)wcnt);
        atomicMin(&sm.mn, tmn);
        atomicMax(&sm.mx, tmx);
    }
    __syncthreads();
    if (tid == 0 && sm.count > 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&p.stats->sum), (unsigned long long)sm.sum);
        atomicAdd(reinterpret_cast<unsigned long long *>(&p.stats->count), (unsigned long long)sm.count);
        atomicMin(&p.stats->mn, sm.mn);
        atomicMax(&p.stats->mx, sm.mx);
    }
}


// Tile-kernel instantiations live in their own translation units (tiles_*.cu, compiled in parallel); the ABI
// unit fetches them through this getter.  family: 0 = FLAVOR 0, 1 = FLAVOR 1 (default), 2 = FLAVOR 2,
// 3 = sparse overrides, 4 = dense table, 5 = wide (words up to 64 symbols), 6 = sparse output, 7 = wide + sparse
// output, 8 = dense table + sparse output, 9 = dense table, wide, 10 = dense table, wide + sparse output.
// qclass: 0/1/2 = register row width 16/24/32 (ignored by the wide families).
typedef void (*nwap_tile_kernel_t)(const nwap_tile_params);
#define NWAP_TILE_FAMILIES 11
nwap_tile_kernel_t nwap_tile_kernel(int family, int qclass);
size_t nwap_tile_smem_bytes(int family, int K = 0);
nwap_tile_kernel_t nwap_tiles_f0f2(int family, int qclass);
nwap_tile_kernel_t nwap_tiles_f1(int qclass);
nwap_tile_kernel_t nwap_tiles_ov(int qclass);
nwap_tile_kernel_t nwap_tiles_tab(int qclass);
nwap_tile_kernel_t nwap_tiles_wide(bool cmp);
nwap_tile_kernel_t nwap_tiles_tabcmp(int qclass);
nwap_tile_kernel_t nwap_tiles_tabwide(bool cmp);
nwap_tile_kernel_t nwap_tiles_cmp(int qclass);
