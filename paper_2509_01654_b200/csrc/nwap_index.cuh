// nwap_index.cuh -- exact 64-bit index arithmetic shared by device and host.
//
// (1) linear edge index <-> (row, col) of the condensed upper triangle
//     (reference triangle.py:43-46, :59-75, :93-112): fp64 closed-form estimate
//     followed by an exact integer bracket correction, evaluated once per row
//     band / per thread, never trusted without the fix-up.
// (2) work-unit enumeration of the tile kernel: the (row, col) plane is cut
//     into bands of NWAP_R rows and strips of NWAP_C columns on an absolute
//     grid; a unit is `group` consecutive bands of one strip.
//
// Compiles as plain C++ (tests/host_emul.cpp) and as CUDA.
#pragma once
#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define NWAP_HD __host__ __device__ __forceinline__
#else
#define NWAP_HD inline
#endif

// Tile geometry (compile-time): a band is R rows, a strip is C columns.
// 320 threads = 10 warps per CTA, two CTAs per SM: the warps of a CTA pull neighbouring chunks of the
// length-sorted strip, so at any moment an SM executes two or three of the 32 length-specialised
// bodies instead of up to twenty (5 CTAs x 4 warps did): the instruction-cache cliff that bounded
// every larger-code variant moves away (profiles/r01h_ab_big_cta.txt).
#ifndef NWAP_THREADS
#define NWAP_THREADS 320       // threads per CTA of the tile kernel
#endif
#ifndef NWAP_R
#define NWAP_R 16
#endif
#define NWAP_C (16 * NWAP_THREADS)   // one aligned uint4 of lengths per thread: 5120 columns
#define NWAP_CHUNK 64          // sorted columns per warp chunk (2 per lane)

// floor(num / m) for |num| <= 12800, 1 <= m <= 255 from one IEEE single-precision division (exact in this
// range: see k_hist_normalized).  Replaces store.py:360's integer floor division on the device.
NWAP_HD int nwap_floor_div_small(int num, int m)
{
#if defined(__CUDA_ARCH__)
    return __float2int_rd(__fdiv_rn((float)num, (float)m));
#else
    return (int)floorf((float)num / (float)m);
#endif
}

NWAP_HD int64_t nwap_before_row(int64_t r, int64_t n) { return (r * (2 * n - r - 1)) >> 1; }

// Row of linear index idx, 0 <= idx < n(n-1)/2.
NWAP_HD int64_t nwap_row_of(int64_t idx, int64_t n)
{
    double z = (double)n - 0.5;
    int64_t r = (int64_t)floor(z - sqrt(z * z - 2.0 * (double)idx));
    if (r < 0) r = 0;
    if (r > n - 2) r = n - 2;
    while (r > 0 && idx < nwap_before_row(r, n)) --r;
    while (idx >= nwap_before_row(r + 1, n)) ++r;
    return r;
}

NWAP_HD int64_t nwap_col_of(int64_t idx, int64_t n, int64_t r)
{
    return r + 1 + (idx - nwap_before_row(r, n));
}

// ---------------------------------------------------------------------------
// Work units.  Bands are aligned to multiples of R, strips to multiples of C
// (absolute), so strip s holds the diagonal of bands [s*C/R, (s+1)*C/R).
// A "group" is `gb` consecutive bands (gb divides C/R, so a group never
// straddles a diagonal strip boundary).  Group g = bands [g*gb, (g+1)*gb);
// its first valid strip is k(g) = (g*gb*R) / C; it owns strips k(g)..S-1.
// Units are enumerated group-major: all strips of group 0, then group 1, ...
// ---------------------------------------------------------------------------
struct nwap_unit_space {
    int64_t n;
    int64_t S;        // number of strips = ceil(n / C)
    int64_t gpk;      // groups per diagonal strip = (C/R) / gb
    int gb;           // bands per group
};

// units before group g (counted from group 0)
NWAP_HD int64_t nwap_units_before_group(const nwap_unit_space &u, int64_t g)
{
    int64_t k = g / u.gpk, rem = g - k * u.gpk;
    // groups in diagonal-strip block kk each own S-kk units
    return u.gpk * (k * u.S - (k * (k - 1)) / 2) + rem * (u.S - k);
}

// decode absolute unit id -> (group, strip)
NWAP_HD void nwap_unit_decode(const nwap_unit_space &u, int64_t t, int64_t *group, int64_t *strip)
{
    // find k with gpk*(k*S - k(k-1)/2) <= t : solve the quadratic in fp64, then fix up.
    double A = (double)(2 * u.S + 1);
    double disc = A * A - 8.0 * ((double)t / (double)u.gpk);
    if (disc < 0.0) disc = 0.0;
    int64_t k = (int64_t)floor((A - sqrt(disc)) * 0.5);
    if (k < 0) k = 0;
    if (k > u.S - 1) k = u.S - 1;
    while (k > 0 && u.gpk * (k * u.S - (k * (k - 1)) / 2) > t) --k;
    while (k + 1 <= u.S - 1 && u.gpk * ((k + 1) * u.S - ((k + 1) * k) / 2) <= t) ++k;
    int64_t rem = t - u.gpk * (k * u.S - (k * (k - 1)) / 2);
    int64_t per = u.S - k;
    int64_t gi = rem / per;
    *group = k * u.gpk + gi;
    *strip = k + (rem - gi * per);
}
