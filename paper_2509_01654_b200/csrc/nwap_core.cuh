// nwap_core.cuh -- the packed Needleman-Wunsch cell update (device + host emulation).
//
// Replaces the inner loops of reference engine.py:159-172 (_nw_batch) for the
// uniform match/mismatch/gap scheme.  Two pairs -- (row word, column word 0) and
// (row word, column word 1) -- live in the two 16-bit halves of every 32-bit
// register ("s16x2").  The rolling score-matrix row stays in registers.
//
// Potential transform (exact integer algebra):
//     H'[i][j] = H[i][j] - (match-gap)*i - gap*j + BIAS
// turns   H[i][j] = max(H[i-1][j-1] + sim, H[i-1][j] + gap, H[i][j-1] + gap)
// into    H'[i][j] = max(H'[i-1][j-1] - e*D,  H'[i-1][j] + u,  H'[i][j-1])
// with e = [a_i != b_j] in {0,1}, D = match - mismatch, u = 2*gap - match,
// boundary H'[0][j] = BIAS, H'[i][0] = BIAS + i*u.
// Per packed cell (2 DP cells) that is
//     e   = VIADDMNMX.U16x2 (row code + column code, min 1)   ALU pipe   (codes: nwap_pack_negb_f; the sum is b - a
//                                                                        mod 2^16, zero iff the symbols are equal)
//     dw  = IMAD            (e * (-D) + diag)        FMA pipe  (packed-safe: halves stay in [0,2^15))
//     cur = VIMNMX3.S16x2   (dw, up_plus_u, left)    ALU pipe
//     upu = IMAD            (cur * 1 + u*65537)      FMA pipe  (next row's up + u)
// i.e. 2 DPX + 2 FMA-pipe issues (FLAVOR 0).  FLAVOR 1 forms up+u with a plain
// 32-bit IADD instead (2 DPX + 1 IMAD + 1 IADD): on B200 the 3-input DPX ops and IMAD
// are half-rate on separate pipes while IADD is full-rate and co-issues with both
// (profiles/r01b_probes.txt).
//
// FLAVOR 2 (needs match >= mismatch) removes two of the four issues.  With the symmetric
// potential H'[i][j] = H[i][j] - gap*(i + j) + BIAS both gap moves cost nothing and every
// boundary cell is BIAS:
//     H'[i][j] = max(H'[i-1][j-1] + C - out,  H'[i-1][j],  H'[i][j-1]),
//     C = match - 2*gap,  out = D * [a_i != b_j],  D = match - mismatch >= 0.
// Symbols are stored multiplied by 256, so (256*a - 256*b) mod 2^16 is 0 when they are equal
// and >= 256 >= D otherwise, and ONE unsigned add-min against the threshold D yields `out`:
//     out = VIADDMNMX.U16x2 (256*a + (-256*b), min D)     ALU pipe (half rate)
//     dw  = IADD3           (diag - out + C*65537)         full rate, co-issues
//     cur = VIMNMX3.S16x2   (dw, up, left)                 ALU pipe (half rate)
// i.e. 3 issues per 2 DP cells, 2 of them on the DPX pipe, which is then the only bound.
//
// All halves stay inside [0, 2^15): |H| <= 128 by the int8 preflight
// (engine.py:72-96), |(match-gap)*i| <= 192, |gap*j| <= 64, |D| <= 256, and
// BIAS = 8192, so 32-bit IMAD never carries between halves and signed/unsigned
// 16-bit max agree.
#pragma once
#include <stdint.h>
#include "nwap_index.cuh"

#ifndef NWAP_BIAS
#define NWAP_BIAS 8192u
#endif
#define NWAP_BIAS2 (NWAP_BIAS | (NWAP_BIAS << 16))

struct nwap_scheme_consts {
    uint32_t neg_delta;   // (uint32)(-(match - mismatch))            IMAD multiplier
    uint32_t u2;          // (uint32)((2*gap - match) * 65537)        32-bit packed addend
    uint32_t u2h;         // uint16(2*gap - match) replicated         per-half addend (VIADDMNMX)
    uint32_t one;         // 1, opaque to the compiler so `cur*one+u2` stays an IMAD
    int32_t alpha;        // row potential per symbol:    match - gap (FLAVOR 0/1), gap (FLAVOR 2)
    int32_t beta;         // column potential per symbol: gap
    uint32_t symmul;      // staged row symbol = a * symmul + symadd:  65537, 0 (FLAVOR 0); -65537, 0x01000100 (FLAVOR 1:
    uint32_t symadd;      // halves 256 - a, see nwap_pack_negb_f); 256*65537, 0 (FLAVOR 2); K, 0 (FLAVOR 3: table row offset)
    uint32_t t2;          // FLAVOR 2: D * 65537, the add-min threshold
    uint32_t c2;          // FLAVOR 2: (match - 2*gap) * 65537
};

// FLAVOR 2 handles match >= mismatch only (D is an unsigned threshold there).
NWAP_HD bool nwap_flavor2_ok(int match, int mismatch) { return match >= mismatch && match - mismatch <= 256; }

NWAP_HD nwap_scheme_consts nwap_make_consts(int match, int mismatch, int gap, int flavor = 1)
{
    nwap_scheme_consts c;
    int u = 2 * gap - match;
    c.neg_delta = (uint32_t)(-(match - mismatch));
    c.u2 = (uint32_t)(u * 65537);
    c.u2h = ((uint32_t)(uint16_t)(int16_t)u) * 0x10001u;
    c.one = 1u;
    c.alpha = match - gap;
    c.beta = gap;
    c.symmul = 65537u;
    c.symadd = 0u;
    if (flavor == 1) { c.symmul = 0u - 65537u; c.symadd = 0x01000100u; }
    c.t2 = 0u;
    c.c2 = 0u;
    if (flavor == 3) {
        // table-driven cell (dense similarity tables): `match` is the table's maximum M; the staged row symbol is
        // the symbol's row offset a*K in the K x K table of E = M - sim (symmul is set to K by the caller)
        c.neg_delta = 0u;
    }
    if (flavor == 2) {
        c.alpha = gap;
        c.u2 = 0u;                                  // every boundary cell H'[i][0] is BIAS
        c.u2h = 0u;
        c.symmul = 256u * 65537u;
        c.t2 = (uint32_t)(match - mismatch) * 65537u;
        c.c2 = (uint32_t)((match - 2 * gap) * 65537);
    }
    return c;
}

NWAP_HD uint32_t nwap_row_code(uint32_t a, const nwap_scheme_consts &sc) { return a * sc.symmul + sc.symadd; }

// ---- DPX intrinsics with host emulation ------------------------------------
#if defined(__CUDA_ARCH__)
#define NWAP_DEV_INTRIN 1
#else
#define NWAP_DEV_INTRIN 0
#endif

NWAP_HD uint32_t nwap_viaddmin_u16x2(uint32_t a, uint32_t b, uint32_t c)
{
#if NWAP_DEV_INTRIN
    return __viaddmin_u16x2(a, b, c);
#else
    uint32_t lo = ((a & 0xffffu) + (b & 0xffffu)) & 0xffffu, hi = ((a >> 16) + (b >> 16)) & 0xffffu;
    uint32_t cl = c & 0xffffu, ch = c >> 16;
    return (lo < cl ? lo : cl) | ((hi < ch ? hi : ch) << 16);
#endif
}

NWAP_HD uint32_t nwap_vimax3_s16x2(uint32_t a, uint32_t b, uint32_t c)
{
#if NWAP_DEV_INTRIN
    return __vimax3_s16x2(a, b, c);
#else
    int16_t al = (int16_t)(a & 0xffffu), ah = (int16_t)(a >> 16);
    int16_t bl = (int16_t)(b & 0xffffu), bh = (int16_t)(b >> 16);
    int16_t cl = (int16_t)(c & 0xffffu), ch = (int16_t)(c >> 16);
    int16_t ml = al > bl ? al : bl; ml = ml > cl ? ml : cl;
    int16_t mh = ah > bh ? ah : bh; mh = mh > ch ? mh : ch;
    return (uint32_t)(uint16_t)ml | ((uint32_t)(uint16_t)mh << 16);
#endif
}

NWAP_HD uint32_t nwap_viaddmax_s16x2(uint32_t a, uint32_t b, uint32_t c)
{
#if NWAP_DEV_INTRIN
    return __viaddmax_s16x2(a, b, c);
#else
    int16_t sl = (int16_t)(uint16_t)((a & 0xffffu) + (b & 0xffffu));
    int16_t sh = (int16_t)(uint16_t)((a >> 16) + (b >> 16));
    int16_t cl = (int16_t)(c & 0xffffu), ch = (int16_t)(c >> 16);
    int16_t ml = sl > cl ? sl : cl, mh = sh > ch ? sh : ch;
    return (uint32_t)(uint16_t)ml | ((uint32_t)(uint16_t)mh << 16);
#endif
}

NWAP_HD uint32_t nwap_vmaxs2(uint32_t a, uint32_t b)
{
#if NWAP_DEV_INTRIN
    return __vmaxs2(a, b);
#else
    return nwap_vimax3_s16x2(a, b, b);
#endif
}

// Negated, packed column symbols: half 0 = -b0[j], half 1 = -b1[j] (mod 2^16),
// so that (a*65537 + nb) has a zero half exactly where the symbols are equal.
NWAP_HD uint32_t nwap_pack_negb(uint32_t b0, uint32_t b1)
{
    return ((0u - b0) & 0xffffu) | ((0u - b1) << 16);
}
// FLAVOR 2 stores symbols times 256 (see the header comment).
// FLAVOR 1 (the default cell) moves the minus sign to the row side so that the column side is a pure byte
// interleave: the column code of symbol b is b + 0xff00 = (b - 256) mod 2^16 -- bytes {b0, 0xff, b1, 0xff}, two byte
// permutes per two columns (nwap_unpack_cols) instead of five shift/mask/negate operations per column -- and the
// staged row code is 256 - a in both halves (a * -65537 + 0x01000100: no borrow, 256 - a >= 1), so that
// (row + column) mod 2^16 = b - a is still zero exactly where the symbols are equal.
template <int FLAVOR>
NWAP_HD uint32_t nwap_pack_negb_f(uint32_t b0, uint32_t b1)
{
    return FLAVOR == 2 ? nwap_pack_negb(b0 << 8, b1 << 8)
         : FLAVOR == 1 ? ((b0 | 0xff00u) | ((b1 | 0xff00u) << 16))
                       : nwap_pack_negb(b0, b1);
}

// One score-matrix row (one symbol of the row word, packed as a*65537) against
// the LB register-resident columns P[1..LB] (P[0] is unused).  d0 = H'[i-1][0],
// left0 = H'[i][0] (both halves).  The cell is software-pipelined: the diagonal
// term of cell j+1 is formed from the OLD P[j] before P[j] is overwritten, so the
// update is in place and the loop over matrix rows needs no register moves and
// no unrolling -- which keeps the per-length code small enough for the
// instruction cache (32 length-specialised bodies live in one kernel).
//
// DOM: the row starts at the matrix border (column 0).  There the boundary value is dominated by the `up` term of
// column 1 -- H'[i][0] = H'[i-1][0] + u <= H'[i-1][1] + u, because the left move is free (H'[i-1][1] >= H'[i-1][0],
// and H'[0][1] = H'[0][0]) -- so cell (i, 1) is max(dw, up + u), left0 is not read, and the staged record only has
// to carry d0 = H'[i-1][0]: no register move per matrix row.
template <int LB, int FLAVOR, bool DOM = false>
NWAP_HD void nwap_dp_row(uint32_t a2, const uint32_t *nb, uint32_t (&P)[LB + 1],
                         uint32_t d0, uint32_t left0, const nwap_scheme_consts &sc)
{
    uint32_t left = left0;
    if (FLAVOR == 2) {
        // d0 arrives with C already added (d0 = BIAS2 + c2, the same for every matrix row)
        uint32_t dw = d0 - nwap_viaddmin_u16x2(a2, nb[0], sc.t2);
#pragma unroll
        for (int j = 1; j <= LB; ++j) {
            uint32_t dw_next = 0;
            if (j < LB) dw_next = P[j] - nwap_viaddmin_u16x2(a2, nb[j], sc.t2) + sc.c2;
            const uint32_t cur = nwap_vimax3_s16x2(dw, P[j], left);
            P[j] = cur;
            left = cur;
            dw = dw_next;
        }
        return;
    }
    uint32_t dw = nwap_viaddmin_u16x2(a2, nb[0], 0x00010001u) * sc.neg_delta + d0;
#pragma unroll
    for (int j = 1; j <= LB; ++j) {
        uint32_t dw_next = 0;
        if (j < LB) dw_next = nwap_viaddmin_u16x2(a2, nb[j], 0x00010001u) * sc.neg_delta + P[j];
        uint32_t cur;
        // up + u: halves stay in [0, 2^15), so a plain 32-bit add/IMAD of u*65537 is a packed add
        const uint32_t upu = FLAVOR == 0 ? P[j] * sc.one + sc.u2 : P[j] + sc.u2;
        cur = (DOM && j == 1) ? nwap_vmaxs2(dw, upu) : nwap_vimax3_s16x2(dw, upu, left);
        P[j] = cur;
        left = cur;
        dw = dw_next;
    }
}

// All la matrix rows of one row word; returns P[] holding matrix row la.
// row_sym2[i] = {row code of a_i, H'[i][0]}: the packed symbol of matrix row i+1 and the boundary value of the row
// ABOVE it (BIAS2 + i*u2, the same for every word: the diagonal term of column 1), fetched together.
struct nwap_sym2 { uint32_t a2, d0; };

// PEEL (FLAVOR 1 only): matrix row 1 is peeled.  Every H'[0][j] is BIAS, so its diagonal term is BIAS - e*D, and
// its up term BIAS + u equals the row's boundary value H'[1][0] the left chain starts from, i.e. it is absorbed:
// H'[1][j] = max(BIAS - e_j*D, H'[1][j-1]) -- three instructions per cell instead of four and no initialisation of
// the rolling row.  Costs 3*LB + 4 instructions of code per body, so only short bodies use it (NWAP_F2_PEEL_MAXLB).
template <int LB, int FLAVOR, bool PEEL = false>
NWAP_HD void nwap_dp_word(const nwap_sym2 *row_sym2, int la, const uint32_t *nb,
                          uint32_t (&P)[LB + 1], const nwap_scheme_consts &sc)
{
    if (PEEL && FLAVOR == 1) {
        const nwap_sym2 *s = row_sym2, *e = row_sym2 + la;
        const nwap_sym2 x0 = *s++;
        uint32_t left = x0.d0 + sc.u2;                      // H'[1][0]
        P[0] = NWAP_BIAS2;
#pragma unroll
        for (int j = 1; j <= LB; ++j) {
            const uint32_t dw = nwap_viaddmin_u16x2(x0.a2, nb[j - 1], 0x00010001u) * sc.neg_delta + NWAP_BIAS2;
            left = nwap_vmaxs2(dw, left);
            P[j] = left;
        }
#pragma unroll 1
        while (s != e) {
            const nwap_sym2 x = *s++;
            nwap_dp_row<LB, FLAVOR, true>(x.a2, nb, P, x.d0, 0u, sc);
        }
        return;
    }
#pragma unroll
    for (int j = 0; j <= LB; ++j) P[j] = NWAP_BIAS2;        // H'[0][j]
    const nwap_sym2 *s = row_sym2, *e = row_sym2 + la;
    if (FLAVOR == 2) {
        const uint32_t d0c = NWAP_BIAS2 + sc.c2;            // H'[i-1][0] + C: every boundary cell is BIAS
#pragma unroll 1
        do {
            const uint32_t a2 = (s++)->a2;
            nwap_dp_row<LB, FLAVOR>(a2, nb, P, d0c, NWAP_BIAS2, sc);
        } while (s != e);
        return;
    }
#pragma unroll 1
    do {                                                    // la >= 1 always
        const nwap_sym2 x = *s++;                           // {symbol, boundary of the row above} in one 8-byte load
        nwap_dp_row<LB, FLAVOR, true>(x.a2, nb, P, x.d0, 0u, sc);
    } while (s != e);
}

// ---- sparse overrides (ScoringScheme.overrides, reference aligner.py:51-65) -----------------
// sim(a, b) = uniform(a, b) + delta(a, b) with delta != 0 for at most NWAP_MAX_OV partners b of any symbol a
// (a itself may be one of them).  For a matrix row whose symbol has partners (p_k, delta_k) the diagonal term is
//     dw = diag - e*D + sum_k delta_k * [b_j == p_k]
//        = diag - e*D - sum_k delta_k * e_k + dsum,   e_k = min(p_k - b_j, 1),  dsum = sum_k delta_k:
// one extra DPX compare + IMAD per partner -- and a constant.  The constant is removed by a ROW potential:
// with G_i = -(dsum of matrix rows 1..i) and H''[i][j] = H'[i][j] + G_i,
//     H''[i][j] = max(H''[i-1][j-1] - e*D - sum_k delta_k*e_k,  H''[i-1][j] + (u - dsum_i),  H''[i][j-1]),
// i.e. the row's `up` addend and its boundary value H''[i][0] = BIAS + i*u + G_i come from the staged row record
// (they did anyway) and the score fix-up of the row word absorbs -G_la.  Rows whose symbol has no partner run the
// plain cell; rows with one / two partners run 6 / 8 instructions per packed cell instead of 4.
#define NWAP_MAX_OV 2
#ifndef NWAP_OV_ONE
#define NWAP_OV_ONE 1               // 1: rows with one partner have their own 6-instruction cell (else they run the 8-instruction one)
#endif
struct nwap_ov_row {                 // one row of the per-symbol override table (32 bytes)
    uint32_t b2[NWAP_MAX_OV];        // partner symbol as a row code (FLAVOR 1: 256 - p in both halves; unused slot: anything)
    uint32_t nd[NWAP_MAX_OV];        // (uint32)(-delta_k)     (unused slot: 0)
    int32_t dsum;                    // sum_k delta_k
    uint32_t count;                  // number of used slots
    uint32_t pad[2];
};
// staged record of one matrix row of an override scheme (one LDS.128) and the per-symbol partner table the
// override rows read on top of it (kept apart so that the staged rows stay small: two CTAs must fit one SM)
struct alignas(16) nwap_sym8 {
    uint32_t a2, left0, ui2, ov;     // row code, H''[i][0], (u - dsum_i) * 65537, 0 = no partner else symbol << 2 | count
};
struct alignas(16) nwap_ov_part {
    uint32_t p0, nd0, p1, nd1;       // partners' row codes and -delta
};

// One score-matrix row with N partners, software-pipelined like nwap_dp_row (the diagonal term of cell j+1 is formed
// from the old P[j] before P[j] is overwritten).
template <int LB, int N>
NWAP_HD void nwap_dp_row_ov(const nwap_sym8 &xr, const nwap_ov_part &y, const uint32_t *nb, uint32_t (&P)[LB + 1],
                            uint32_t d0, const nwap_scheme_consts &sc)
{
    struct { uint32_t a2, left0, ui2, p0, nd0, p1, nd1; } x = {xr.a2, xr.left0, xr.ui2, y.p0, y.nd0, y.p1, y.nd1};
    uint32_t left = x.left0;
    uint32_t dw = nwap_viaddmin_u16x2(x.a2, nb[0], 0x00010001u) * sc.neg_delta + d0;
    dw = nwap_viaddmin_u16x2(x.p0, nb[0], 0x00010001u) * x.nd0 + dw;
    if (N > 1) dw = nwap_viaddmin_u16x2(x.p1, nb[0], 0x00010001u) * x.nd1 + dw;
#pragma unroll
    for (int j = 1; j <= LB; ++j) {
        uint32_t dw_next = 0;
        if (j < LB) {
            dw_next = nwap_viaddmin_u16x2(x.a2, nb[j], 0x00010001u) * sc.neg_delta + P[j];
            dw_next = nwap_viaddmin_u16x2(x.p0, nb[j], 0x00010001u) * x.nd0 + dw_next;
            if (N > 1) dw_next = nwap_viaddmin_u16x2(x.p1, nb[j], 0x00010001u) * x.nd1 + dw_next;
        }
        const uint32_t cur = nwap_vimax3_s16x2(dw, P[j] + x.ui2, left);
        P[j] = cur;
        left = cur;
        dw = dw_next;
    }
}

template <int LB, int FLAVOR>
NWAP_HD void nwap_dp_word_ov(const nwap_sym8 *rec, int la, const uint32_t *nb, uint32_t (&P)[LB + 1],
                             const nwap_scheme_consts &sc, const nwap_ov_part *parts)
{
#pragma unroll
    for (int j = 0; j <= LB; ++j) P[j] = NWAP_BIAS2;
    uint32_t d0 = NWAP_BIAS2;
    const nwap_sym8 *s = rec, *e = rec + la;
    // the record of the next matrix row is fetched a row ahead: the dispatch on its partner count would otherwise
    // wait for the load at every row (rec[la] is readable: the staged rows hold one record more than the longest word)
#pragma unroll 1
    do {
        const nwap_sym8 x = *s++;
        if (x.ov == 0) nwap_dp_row<LB, FLAVOR>(x.a2, nb, P, d0, x.left0, sc);
        else {
            const nwap_ov_part y = parts[x.ov >> 2];
#if NWAP_OV_ONE
            if ((x.ov & 3u) == 1u) nwap_dp_row_ov<LB, 1>(x, y, nb, P, d0, sc);
            else
#endif
            nwap_dp_row_ov<LB, 2>(x, y, nb, P, d0, sc);
        }
        d0 = x.left0;
    } while (s != e);
}

// Staged records of one row word (a[0..la)): row codes, partners, and the row potential folded into the boundary
// values and `up` addends.  Returns sum_i dsum(a_i) = -G_la, which the caller adds to the row word's score fix-up.
NWAP_HD int nwap_stage_row_ov(const uint8_t *a, int la, const nwap_ov_row *tab, int K, const nwap_scheme_consts &sc,
                              nwap_sym8 *rec)
{
    const int u = (int)(int16_t)(sc.u2h & 0xffffu);
    int gsum = 0;
    for (int i = 0; i < la; ++i) {
        const uint32_t sym = a[i];
        nwap_sym8 x;
        x.a2 = nwap_row_code(sym, sc);
        x.ov = 0;
        int ds = 0;
        if ((int)sym < K && tab[sym].count) {
            x.ov = (sym << 2) | tab[sym].count;
            ds = tab[sym].dsum;
        }
        gsum += ds;
        x.left0 = NWAP_BIAS2 + (uint32_t)((i + 1) * u - gsum) * 65537u;
        x.ui2 = (uint32_t)(u - ds) * 65537u;
        rec[i] = x;
    }
    return gsum;
}

// Host-side construction of the override table from a dense K x K similarity table
// (reference engine.py:110-117).  Returns false when some symbol has more than NWAP_MAX_OV
// partners (the scheme then goes to the table-driven cell or the generic kernel).
inline bool nwap_build_ov_table(const int8_t *sim, int K, int match, int mismatch, nwap_ov_row *out)
{
    for (int a = 0; a < K; ++a) {
        nwap_ov_row r;
        for (int k = 0; k < NWAP_MAX_OV; ++k) { r.b2[k] = 0; r.nd[k] = 0; }
        r.pad[0] = r.pad[1] = 0;
        int cnt = 0, dsum = 0;
        for (int b = 0; b < K; ++b) {
            const int delta = (int)sim[a * K + b] - (a == b ? match : mismatch);
            if (delta == 0) continue;
            if (cnt == NWAP_MAX_OV) return false;
            r.b2[cnt] = 0x01000100u - (uint32_t)b * 65537u;
            r.nd[cnt] = (uint32_t)(-delta);
            dsum += delta;
            ++cnt;
        }
        r.dsum = dsum;
        r.count = (uint32_t)cnt;
        out[a] = r;
    }
    return true;
}

// ---- dense similarity tables (FLAVOR 3): sim(a, b) = M - E[a][b] with M the table's maximum and E a K x K
// uint8 table in shared memory.  With match := M the potentials of FLAVOR 1 carry over and the diagonal term is
//     dw = diag - (E[a_i][b0_j] | E[a_i][b1_j] << 16)
// (non-negative halves subtracted from biased halves: no borrow crosses).  Two byte loads per packed cell replace
// the compare + multiply; c0/c1 hold the lane's column symbols as byte offsets.
template <int LB, bool DOM = true>
NWAP_HD void nwap_dp_row_tab(uint32_t rowoff, const uint32_t *c0, const uint32_t *c1, uint32_t (&P)[LB + 1],
                             uint32_t d0, const nwap_scheme_consts &sc, const uint8_t *etab, uint32_t left0 = 0u)
{
    const uint8_t *row = etab + rowoff;
    uint32_t left = left0;                                  // DOM (matrix border): column 1's boundary is dominated (nwap_dp_row)
    uint32_t dw = d0 - ((uint32_t)row[c0[0]] | ((uint32_t)row[c1[0]] << 16));
#pragma unroll
    for (int j = 1; j <= LB; ++j) {
        uint32_t dw_next = 0;
        if (j < LB) dw_next = P[j] - ((uint32_t)row[c0[j]] | ((uint32_t)row[c1[j]] << 16));
        const uint32_t cur = (DOM && j == 1) ? nwap_vmaxs2(dw, P[j] + sc.u2) : nwap_vimax3_s16x2(dw, P[j] + sc.u2, left);
        P[j] = cur;
        left = cur;
        dw = dw_next;
    }
}

template <int LB>
NWAP_HD void nwap_dp_word_tab(const nwap_sym2 *row_sym2, int la, const uint32_t *c0, const uint32_t *c1,
                              uint32_t (&P)[LB + 1], const nwap_scheme_consts &sc, const uint8_t *etab)
{
#pragma unroll
    for (int j = 0; j <= LB; ++j) P[j] = NWAP_BIAS2;
    const nwap_sym2 *s = row_sym2, *e = row_sym2 + la;
#pragma unroll 1
    do {
        const nwap_sym2 x = *s++;
        nwap_dp_row_tab<LB>(x.a2, c0, c1, P, x.d0, sc, etab);
    } while (s != e);
}

// ---- column words longer than the register-resident row (24 < length <= 64) -------------------
// The int8 preflight admits words of up to 64 symbols for gap -1 -- the paper's own scheme
// (1,-1,-1), reference engine.py:83-90 -- but a 64-column rolling row plus 64 packed symbols
// does not fit the register budget of two 320-thread CTAs per SM.  Such chunks are scored in
// blocks of NWAP_WB columns: block k is the same software-pipelined row update at register
// width NWAP_WB whose left boundary is not the matrix border but column NWAP_WB*k of the same
// matrix row, saved by block k-1 (one 32-bit word per matrix row per lane, `save`).  The
// recurrence H'[i][j] = max(H'[i-1][j-1] - e*D, H'[i-1][j] + u, H'[i][j-1]) holds at every j,
// so (d0, left0) = (H'[i-1][WB*k], H'[i][WB*k]) is all a block needs from its left neighbour.
// b0 / b1: the two column words' symbols, readable (padding included) up to NWAP_WB*nblk bytes.
// Returns the packed H'[la][l0] | H'[la][l1] << 16.
#define NWAP_WB 16
#define NWAP_MAXLEN_WIDE 64

NWAP_HD void nwap_load_block_negb(const uint8_t *b0, const uint8_t *b1, uint32_t (&nb)[NWAP_WB])
{
#if defined(__CUDA_ARCH__)
    const uint4 x = __ldg(reinterpret_cast<const uint4 *>(b0));
    const uint4 y = __ldg(reinterpret_cast<const uint4 *>(b1));
    const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int j = 0; j < NWAP_WB; ++j)
        nb[j] = nwap_pack_negb_f<1>((xw[j >> 2] >> (8 * (j & 3))) & 0xffu, (yw[j >> 2] >> (8 * (j & 3))) & 0xffu);
#else
    for (int j = 0; j < NWAP_WB; ++j) nb[j] = nwap_pack_negb_f<1>(b0[j], b1[j]);
#endif
}

NWAP_HD uint32_t nwap_dp_blocks(const nwap_sym2 *row_sym2, int la, const uint8_t *b0, const uint8_t *b1, int nblk,
                                int l0, int l1, const nwap_scheme_consts &sc, uint32_t *save)
{
    uint32_t lo = 0, hi = 0;
    for (int blk = 0; blk < nblk; ++blk) {
        uint32_t nb[NWAP_WB];
        nwap_load_block_negb(b0 + NWAP_WB * blk, b1 + NWAP_WB * blk, nb);
        uint32_t P[NWAP_WB + 1];
#pragma unroll
        for (int j = 0; j <= NWAP_WB; ++j) P[j] = NWAP_BIAS2;      // H'[0][j]
        uint32_t d0 = NWAP_BIAS2;                                  // H'[0][WB*blk]
#pragma unroll 1
        for (int i = 0; i < la; ++i) {
            const nwap_sym2 x = row_sym2[i];
            const uint32_t left0 = blk == 0 ? x.d0 + sc.u2 : save[i]; // H'[i+1][WB*blk]
            nwap_dp_row<NWAP_WB, 1>(x.a2, nb, P, d0, left0, sc);
            d0 = left0;
            save[i] = P[NWAP_WB];                                  // H'[i+1][WB*(blk+1)] for the next block
        }
        const int j0 = l0 - NWAP_WB * blk, j1 = l1 - NWAP_WB * blk;
#pragma unroll
        for (int j = 1; j <= NWAP_WB; ++j) {
            if (j == j0) lo = P[j] & 0xffffu;
            if (j == j1) hi = P[j] & 0xffff0000u;
        }
    }
    return lo | hi;
}

// The same block-wise scoring with the table-driven cell (FLAVOR 3: row_sym2[i].a2 is the row offset a_i * K in the
// K x K table of M - sim): override schemes over words of up to 64 symbols stay on the packed kernel.
NWAP_HD uint32_t nwap_dp_blocks_tab(const nwap_sym2 *row_sym2, int la, const uint8_t *b0, const uint8_t *b1, int nblk,
                                    int l0, int l1, const nwap_scheme_consts &sc, uint32_t *save, const uint8_t *etab)
{
    uint32_t lo = 0, hi = 0;
    for (int blk = 0; blk < nblk; ++blk) {
        uint32_t c0[NWAP_WB], c1[NWAP_WB];
#if defined(__CUDA_ARCH__)
        {
            const uint4 x = __ldg(reinterpret_cast<const uint4 *>(b0 + NWAP_WB * blk));
            const uint4 y = __ldg(reinterpret_cast<const uint4 *>(b1 + NWAP_WB * blk));
            const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int j = 0; j < NWAP_WB; ++j) {
                c0[j] = (xw[j >> 2] >> (8 * (j & 3))) & 0xffu;
                c1[j] = (yw[j >> 2] >> (8 * (j & 3))) & 0xffu;
            }
        }
#else
        for (int j = 0; j < NWAP_WB; ++j) { c0[j] = b0[NWAP_WB * blk + j]; c1[j] = b1[NWAP_WB * blk + j]; }
#endif
        uint32_t P[NWAP_WB + 1];
#pragma unroll
        for (int j = 0; j <= NWAP_WB; ++j) P[j] = NWAP_BIAS2;      // H'[0][j]
        uint32_t d0 = NWAP_BIAS2;                                  // H'[0][WB*blk]
#pragma unroll 1
        for (int i = 0; i < la; ++i) {
            const nwap_sym2 x = row_sym2[i];
            const uint32_t left0 = blk == 0 ? x.d0 + sc.u2 : save[i]; // H'[i+1][WB*blk]
            nwap_dp_row_tab<NWAP_WB, false>(x.a2, c0, c1, P, d0, sc, etab, left0);
            d0 = left0;
            save[i] = P[NWAP_WB];
        }
        const int j0 = l0 - NWAP_WB * blk, j1 = l1 - NWAP_WB * blk;
#pragma unroll
        for (int j = 1; j <= NWAP_WB; ++j) {
            if (j == j0) lo = P[j] & 0xffffu;
            if (j == j1) hi = P[j] & 0xffff0000u;
        }
    }
    return lo | hi;
}

// Whole pair-of-pairs DP for one row word; returns the packed H' values at
// (la, lb0) in the low half and (la, lb1) in the high half.  Used by the host
// emulation test; the tile kernel calls nwap_dp_word directly.
template <int LB, int FLAVOR, bool PEEL = false>
NWAP_HD uint32_t nwap_dp_pair(const nwap_sym2 *row_sym2, int la, const uint32_t (&nb)[LB],
                              int lb0, int lb1, const nwap_scheme_consts &sc)
{
    uint32_t P[LB + 1];
    nwap_dp_word<LB, FLAVOR, PEEL>(row_sym2, la, nb, P, sc);
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int j = 1; j <= LB; ++j) {
        if (j == lb0) lo = P[j] & 0xffffu;
        if (j == lb1) hi = P[j] >> 16;
    }
    return lo | (hi << 16);
}

// H'[la][lb] (one half, biased) -> true score.
NWAP_HD int nwap_unbias(uint32_t half, int la, int lb, const nwap_scheme_consts &sc)
{
    return (int)half - (int)NWAP_BIAS + sc.alpha * la + sc.beta * lb;
}
