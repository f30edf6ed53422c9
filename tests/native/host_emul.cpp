// tests/native/host_emul.cpp -- compiles the device headers as plain C++ so the
// packed-recurrence algebra and the index/unit arithmetic can be checked on a
// CPU against the oracle (tests/test_core_emul.py).  Test infrastructure only.
#include <stdint.h>
#include <string.h>
#include "nwap_index.cuh"
#include "nwap_core.cuh"

template <int LB, int FLAVOR, bool PEEL = false>
static uint32_t run_pair(const uint8_t *a, int la, const uint8_t *b0, int lb0,
                         const uint8_t *b1, int lb1, const nwap_scheme_consts &sc)
{
    nwap_sym2 row2[256];
    for (int i = 0; i < la; ++i) {
        row2[i].a2 = nwap_row_code(a[i], sc);
        row2[i].d0 = NWAP_BIAS2 + (uint32_t)i * sc.u2;

    }
    uint32_t nb[LB];
    for (int j = 0; j < LB; ++j)
        nb[j] = nwap_pack_negb_f<FLAVOR>(j < lb0 ? b0[j] : 0u, j < lb1 ? b1[j] : 0u);
    return nwap_dp_pair<LB, FLAVOR, PEEL>(row2, la, nb, lb0, lb1, sc);
}

template <int FLAVOR, bool PEEL = false>
static uint32_t dispatch(int LB, const uint8_t *a, int la, const uint8_t *b0, int lb0,
                         const uint8_t *b1, int lb1, const nwap_scheme_consts &sc)
{
    switch (LB) {
#define CASE(n) case n: return run_pair<n, FLAVOR, PEEL>(a, la, b0, lb0, b1, lb1, sc);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
        CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23) CASE(24)
        CASE(25) CASE(26) CASE(27) CASE(28) CASE(29) CASE(30) CASE(31) CASE(32)
#undef CASE
    }
    return 0;
}

template <int LB>
static uint32_t run_pair_ov(const uint8_t *a, int la, const uint8_t *b0, int lb0, const uint8_t *b1, int lb1,
                            const nwap_scheme_consts &sc, const nwap_ov_row *tab, int K, int *gsum)
{
    nwap_sym8 rec[256];
    *gsum = nwap_stage_row_ov(a, la, tab, K, sc, rec);
    uint32_t nb[LB];
    for (int j = 0; j < LB; ++j) nb[j] = nwap_pack_negb_f<1>(j < lb0 ? b0[j] : 0u, j < lb1 ? b1[j] : 0u);
    static nwap_ov_part parts[256];
    for (int k = 0; k < K; ++k) { parts[k].p0 = tab[k].b2[0]; parts[k].nd0 = tab[k].nd[0]; parts[k].p1 = tab[k].b2[1]; parts[k].nd1 = tab[k].nd[1]; }
    uint32_t P[LB + 1];
    nwap_dp_word_ov<LB, 1>(rec, la, nb, P, sc, parts);
    uint32_t lo = 0, hi = 0;
    for (int j = 1; j <= LB; ++j) {
        if (j == lb0) lo = P[j] & 0xffffu;
        if (j == lb1) hi = P[j] >> 16;
    }
    return lo | (hi << 16);
}

template <int LB>
static uint32_t run_pair_tab(const uint8_t *a, int la, const uint8_t *b0, int lb0, const uint8_t *b1, int lb1,
                             const nwap_scheme_consts &sc, const uint8_t *etab, int K)
{
    nwap_sym2 row2[256];
    for (int i = 0; i < la; ++i) {
        row2[i].a2 = (uint32_t)a[i] * (uint32_t)K;
        row2[i].d0 = NWAP_BIAS2 + (uint32_t)i * sc.u2;
    }
    uint32_t c0[LB], c1[LB];
    for (int j = 0; j < LB; ++j) { c0[j] = j < lb0 ? b0[j] : 0u; c1[j] = j < lb1 ? b1[j] : 0u; }
    uint32_t P[LB + 1];
    nwap_dp_word_tab<LB>(row2, la, c0, c1, P, sc, etab);
    uint32_t lo = 0, hi = 0;
    for (int j = 1; j <= LB; ++j) {
        if (j == lb0) lo = P[j] & 0xffffu;
        if (j == lb1) hi = P[j] >> 16;
    }
    return lo | (hi << 16);
}

extern "C" {

// Dense-table mode: sim is a K x K int8 table; E = max - sim.
int emul_pair_scores_tab(int LB, const uint8_t *a, int la, const uint8_t *b0, int lb0, const uint8_t *b1, int lb1,
                         const int8_t *sim, int K, int gap, int *s0, int *s1)
{
    if (LB < 1 || LB > 32 || lb0 > LB || lb1 > LB || la < 1 || K > 128) return -1;
    static uint8_t etab[128 * 128];
    int M = -128;
    for (int i = 0; i < K * K; ++i) M = sim[i] > M ? sim[i] : M;
    for (int i = 0; i < K * K; ++i) etab[i] = (uint8_t)(M - sim[i]);
    nwap_scheme_consts sc = nwap_make_consts(M, M, gap, 3);
    uint32_t v = 0;
    switch (LB) {
#define CASE(n) case n: v = run_pair_tab<n>(a, la, b0, lb0, b1, lb1, sc, etab, K); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
        CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23) CASE(24)
        CASE(25) CASE(26) CASE(27) CASE(28) CASE(29) CASE(30) CASE(31) CASE(32)
#undef CASE
    }
    *s0 = nwap_unbias(v & 0xffffu, la, lb0, sc);
    *s1 = nwap_unbias(v >> 16, la, lb1, sc);
    return 0;
}

// Sparse-override mode: sim is a dense K x K int8 table; returns -2 when it is not sparse enough.
int emul_pair_scores_ov(int LB, const uint8_t *a, int la, const uint8_t *b0, int lb0, const uint8_t *b1, int lb1,
                        const int8_t *sim, int K, int match, int mismatch, int gap, int *s0, int *s1)
{
    if (LB < 1 || LB > 32 || lb0 > LB || lb1 > LB || la < 1 || K > 256) return -1;
    static nwap_ov_row tab[256];
    if (!nwap_build_ov_table(sim, K, match, mismatch, tab)) return -2;
    nwap_scheme_consts sc = nwap_make_consts(match, mismatch, gap);
    uint32_t v = 0;
    int gsum = 0;
    switch (LB) {
#define CASE(n) case n: v = run_pair_ov<n>(a, la, b0, lb0, b1, lb1, sc, tab, K, &gsum); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
        CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23) CASE(24)
        CASE(25) CASE(26) CASE(27) CASE(28) CASE(29) CASE(30) CASE(31) CASE(32)
#undef CASE
    }
    *s0 = nwap_unbias(v & 0xffffu, la, lb0, sc) + gsum;          // the row potential's share of the fix-up
    *s1 = nwap_unbias(v >> 16, la, lb1, sc) + gsum;
    return 0;
}

// Words of up to 64 symbols: the block-wise path of the tile kernel (nwap_dp_blocks).
int emul_pair_scores_wide(const uint8_t *a, int la, const uint8_t *b0, int lb0, const uint8_t *b1, int lb1,
                          int match, int mismatch, int gap, int *s0, int *s1)
{
    if (la < 1 || la > NWAP_MAXLEN_WIDE || lb0 < 1 || lb1 < 1 || lb0 > NWAP_MAXLEN_WIDE || lb1 > NWAP_MAXLEN_WIDE) return -1;
    nwap_scheme_consts sc = nwap_make_consts(match, mismatch, gap, 1);
    nwap_sym2 row2[NWAP_MAXLEN_WIDE + 1];
    for (int i = 0; i < la; ++i) {
        row2[i].a2 = nwap_row_code(a[i], sc);
        row2[i].d0 = NWAP_BIAS2 + (uint32_t)i * sc.u2;
    }
    uint8_t p0[NWAP_MAXLEN_WIDE + NWAP_WB] = {0}, p1[NWAP_MAXLEN_WIDE + NWAP_WB] = {0};
    memcpy(p0, b0, lb0);
    memcpy(p1, b1, lb1);
    const int LB = lb0 > lb1 ? lb0 : lb1;
    uint32_t save[NWAP_MAXLEN_WIDE + 1];
    const uint32_t v = nwap_dp_blocks(row2, la, p0, p1, (LB + NWAP_WB - 1) / NWAP_WB, lb0, lb1, sc, save);
    *s0 = nwap_unbias(v & 0xffffu, la, lb0, sc);
    *s1 = nwap_unbias(v >> 16, la, lb1, sc);
    return 0;
}

// Words of up to 64 symbols under a dense similarity table: the block-wise path with the table-driven cell
// (nwap_dp_blocks_tab; rows carry the table row offset a * K).
int emul_pair_scores_wide_tab(const uint8_t *a, int la, const uint8_t *b0, int lb0, const uint8_t *b1, int lb1,
                              const int8_t *sim, int K, int gap, int *s0, int *s1)
{
    if (la < 1 || la > NWAP_MAXLEN_WIDE || lb0 < 1 || lb1 < 1 || lb0 > NWAP_MAXLEN_WIDE || lb1 > NWAP_MAXLEN_WIDE || K > 128) return -1;
    static uint8_t etab[128 * 128];
    int M = -128;
    for (int i = 0; i < K * K; ++i) M = sim[i] > M ? sim[i] : M;
    for (int i = 0; i < K * K; ++i) etab[i] = (uint8_t)(M - sim[i]);
    nwap_scheme_consts sc = nwap_make_consts(M, M, gap, 3);
    sc.symmul = (uint32_t)K;
    nwap_sym2 row2[NWAP_MAXLEN_WIDE + 1];
    for (int i = 0; i < la; ++i) {
        row2[i].a2 = nwap_row_code(a[i], sc);
        row2[i].d0 = NWAP_BIAS2 + (uint32_t)i * sc.u2;
    }
    uint8_t p0[NWAP_MAXLEN_WIDE + NWAP_WB] = {0}, p1[NWAP_MAXLEN_WIDE + NWAP_WB] = {0};
    memcpy(p0, b0, lb0);
    memcpy(p1, b1, lb1);
    const int LB = lb0 > lb1 ? lb0 : lb1;
    uint32_t save[NWAP_MAXLEN_WIDE + 1];
    const uint32_t v = nwap_dp_blocks_tab(row2, la, p0, p1, (LB + NWAP_WB - 1) / NWAP_WB, lb0, lb1, sc, save, etab);
    *s0 = nwap_unbias(v & 0xffffu, la, lb0, sc);
    *s1 = nwap_unbias(v >> 16, la, lb1, sc);
    return 0;
}

// Scores (a vs b0) and (a vs b1) with the packed recurrence at register width LB.
int emul_pair_scores(int flavor, int LB, const uint8_t *a, int la, const uint8_t *b0, int lb0,
                     const uint8_t *b1, int lb1, int match, int mismatch, int gap,
                     int *s0, int *s1)
{
    if (LB < 1 || LB > 32 || lb0 > LB || lb1 > LB || la < 1 || lb0 < 1 || lb1 < 1) return -1;
    if (flavor == 2 && !nwap_flavor2_ok(match, mismatch)) return -3;
    // flavor 11: the default cell (FLAVOR 1) with the peeled first matrix row
    nwap_scheme_consts sc = nwap_make_consts(match, mismatch, gap, flavor == 11 ? 1 : flavor);
    uint32_t v = flavor == 0 ? dispatch<0>(LB, a, la, b0, lb0, b1, lb1, sc)
               : flavor == 1 ? dispatch<1>(LB, a, la, b0, lb0, b1, lb1, sc)
               : flavor == 11 ? dispatch<1, true>(LB, a, la, b0, lb0, b1, lb1, sc)
                             : dispatch<2>(LB, a, la, b0, lb0, b1, lb1, sc);
    *s0 = nwap_unbias(v & 0xffffu, la, lb0, sc);
    *s1 = nwap_unbias(v >> 16, la, lb1, sc);
    return 0;
}

int64_t emul_row_of(int64_t idx, int64_t n) { return nwap_row_of(idx, n); }
int64_t emul_col_of(int64_t idx, int64_t n, int64_t r) { return nwap_col_of(idx, n, r); }

int64_t emul_units_before_group(int64_t n, int gb, int64_t g)
{
    nwap_unit_space u; u.n = n; u.S = (n + NWAP_C - 1) / NWAP_C; u.gb = gb; u.gpk = (NWAP_C / NWAP_R) / gb;
    return nwap_units_before_group(u, g);
}

void emul_unit_decode(int64_t n, int gb, int64_t t, int64_t *group, int64_t *strip)
{
    nwap_unit_space u; u.n = n; u.S = (n + NWAP_C - 1) / NWAP_C; u.gb = gb; u.gpk = (NWAP_C / NWAP_R) / gb;
    nwap_unit_decode(u, t, group, strip);
}

int emul_floor_div_small(int num, int m) { return nwap_floor_div_small(num, m); }

int emul_geometry(int *R, int *C, int *chunk) { *R = NWAP_R; *C = NWAP_C; *chunk = NWAP_CHUNK; return 0; }
}
