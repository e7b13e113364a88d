// prngd_device.cuh -- __device__ building blocks of the PRNGD path (sm_100a).
// Product code; written independently of oracle/ (shares nothing with it).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "prngd_internal.h"

namespace prngd {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;      // SplitMix64 increment
constexpr double kBelowOne = 0x1.fffffffffffffp-1;       // 1 - 2^-53, R11 clamp value

// ---- S1: stream init (R6) --------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix_finalize(uint64_t v) {
    v ^= v >> 30;
    v *= 0xBF58476D1CE4E5B9ull;
    v ^= v >> 27;
    v *= 0x94D049BB133111EBull;
    return v ^ (v >> 31);
}

struct Xs128 {
    uint32_t x, y, z, w;
};

// Global stream s starts from SplitMix64(seed) outputs #2s and #2s+1 (counter addressed).
__device__ __forceinline__ Xs128 stream_start(uint64_t seed, uint64_t s) {
    const uint64_t lo = splitmix_finalize(seed + (2 * s + 1) * kGamma);
    const uint64_t hi = splitmix_finalize(seed + (2 * s + 2) * kGamma);
    Xs128 r;
    r.x = (uint32_t)lo;
    r.y = (uint32_t)(lo >> 32);
    r.z = (uint32_t)hi;
    r.w = (uint32_t)(hi >> 32);
    return r;
}

// ---- NEXT-2: MRG32k3a (L'Ecuyer 1999), integer form -------------------------------------------
constexpr uint32_t kM1 = 4294967087u;  // 2^32 - 209
constexpr uint32_t kM2 = 4294944443u;  // 2^32 - 22853

struct Mrg32k3a {
    uint32_t s0, s1, s2;  // component 1, oldest first
    uint32_t t0, t1, t2;  // component 2
};

// One MRG32k3a output u in [1, m1] (R21): x_n = 1403580 x_{n-2} - 810728 x_{n-3} mod m1,
// y_n = 527612 y_{n-1} - 1370589 y_{n-3} mod m2, u = (x_n - y_n) mod m1 with 0 -> m1.  The
// negative terms are written as +a (m - s), so each combination t is a nonnegative u64 < 2^54;
// t mod (2^32 - c) folds the high word with 2^32 = c (mod m):
//   m1 (c = 209):   one fold leaves r < 2^32 + 2^28.8 < 2 m1
//   m2 (c = 22853): two folds leave r < 2^32 + 2^17.8 < 2 m2
// and the final r - m, when r >= m, is the 32-bit sum lo(r) + c (wrapping when hi(r) = 0).
// component 1: x_n = (1403580 x_{n-2} - 810728 x_{n-3}) mod m1 from (x_{n-2}, x_{n-3});
// fold in 32-bit halves (hi * 209 < 2^32, so the sum carries at most once)
__device__ __forceinline__ uint32_t mrg_c1(uint32_t xm2, uint32_t xm3) {
    const uint64_t t1 = 1403580ull * xm2 + 810728ull * (kM1 - xm3);
    const uint32_t h1 = (uint32_t)(t1 >> 32), l1 = (uint32_t)t1;
    const uint32_t f1 = l1 + h1 * 209u;
    return (f1 < l1 || f1 >= kM1) ? f1 + 209u : f1;
}
// component 2: y_n = (527612 y_{n-1} - 1370589 y_{n-3}) mod m2 from (y_{n-1}, y_{n-3});
// first fold kept as (hi, lo) 32-bit words, second fold as above
__device__ __forceinline__ uint32_t mrg_c2(uint32_t ym1, uint32_t ym3) {
    const uint64_t t2 = 527612ull * ym1 + 1370589ull * (kM2 - ym3);
    const uint32_t h2 = (uint32_t)(t2 >> 32), l2 = (uint32_t)t2;
    const uint32_t g_lo = l2 + h2 * 22853u;
    const uint32_t g_hi = __umulhi(h2, 22853u) + (g_lo < l2 ? 1u : 0u);
    const uint32_t f2 = g_lo + g_hi * 22853u;
    return (f2 < g_lo || f2 >= kM2) ? f2 + 22853u : f2;
}
// u = (x_n - y_n) mod m1 with 0 reported as m1
__device__ __forceinline__ uint32_t mrg_combine(uint32_t p1, uint32_t p2) {
    const uint32_t z = p1 - p2;  // wraps when p1 <= p2: then p1 - p2 + m1 = z - 209 (mod 2^32)
    return p1 > p2 ? z : z - 209u;
}

__device__ __forceinline__ uint32_t mrg_next(Mrg32k3a &m) {
    const uint32_t p1 = mrg_c1(m.s1, m.s0);
    m.s0 = m.s1;
    m.s1 = m.s2;
    m.s2 = p1;
    const uint32_t p2 = mrg_c2(m.t2, m.t0);
    m.t0 = m.t1;
    m.t1 = m.t2;
    m.t2 = p2;
    return mrg_combine(p1, p2);
}

// The same recurrences in binary64, on balanced representatives: every product and sum below
// is an integer < 2^53, so each operation is exact.  k = p * (1/m) rounded to an integer by the
// 2^52 + 2^51 shift (nearest, up to the rounding of p * (1/m), which only moves r by one m
// near a half-integer quotient), r = p - k m.  r is congruent to the integer recurrence's value
// and |r| <= m/2 + 2 < 2^31, so no correction is needed between draws: with |x| < 2^31 (or a
// canonical x < 2^32 in one operand, the stream start) |1403580 x - 810728 x'| and
// |527612 y - 1370589 y'| stay below 8e15 < 2^53.  The canonical values are taken only when a
// draw is combined (mrg_combined_b, integer).  m and 1/m come from the kernel parameters, so
// the FMAs read them from the constant bank.
constexpr double kRoundShift = 6755399441055744.0;  // 2^52 + 2^51
// PRNGD_MRG_FLOOR (default): k = floor(p * (1/m)) instead of the nearest integer, by the same
// shift added in round-down mode.  Then r = p - k m lies in [0, m]: with |p| <= 1403580 m1 <
// 6.1e15 the product p * RN(1/m) differs from p / m by less than 1.6e-10 < 1/m, so the floor is
// floor(p / m) except when m divides p exactly, where it may come out one lower and give r = m
// (= 0 mod m).  Values in [0, m] keep every product below 2^53 (the two terms of a recurrence
// have opposite signs: |p| <= max(a, a') m < 6.1e15), so no correction is ever needed between
// draws, and the combination takes r itself as the canonical value (component 2 maps m2 to 0
// with one min; component 1's m1 is handled by mrg_combine_m1 as 0).
#ifndef PRNGD_MRG_FLOOR
#define PRNGD_MRG_FLOOR 1
#endif
__device__ __forceinline__ double mrg_modb(double p, double m, double inv_m) {
#if PRNGD_MRG_FLOOR
    const double k = __dsub_rn(__fma_rd(p, inv_m, kRoundShift), kRoundShift);
#else
    const double k = __dsub_rn(__fma_rn(p, inv_m, kRoundShift), kRoundShift);
#endif
    return __fma_rn(-k, m, p);
}
__device__ __forceinline__ double mrg_c1d(double xm2, double xm3, double m1, double inv_m1) {
    return mrg_modb(__fma_rn(1403580.0, xm2, -__dmul_rn(810728.0, xm3)), m1, inv_m1);
}
__device__ __forceinline__ double mrg_c2d(double ym1, double ym3, double m2, double inv_m2) {
    return mrg_modb(__fma_rn(527612.0, ym1, -__dmul_rn(1370589.0, ym3)), m2, inv_m2);
}
// u - 1 for u = (x_n - y_n) mod m1 in [1, m1] (mrg_combine), as one three-input add
__device__ __forceinline__ uint32_t mrg_combine_m1(uint32_t p1, uint32_t p2) {
    const uint32_t z = p1 - p2 - 1u;
    return p1 > p2 ? z : z - 209u;
}
// u - 1 from p1 = x_n (mod m1), p2 = y_n (mod m2): balanced representatives, or with
// PRNGD_MRG_FLOOR values in [0, m] (see mrg_modb)
__device__ __forceinline__ uint32_t mrg_canon1(double p1) {
#if PRNGD_MRG_FLOOR
    return __double2uint_rz(p1);  // exact; m1 (= 0 mod m1) is handled by mrg_combine_m1
#else
    const int32_t i1 = __double2int_rz(p1);
    return i1 < 0 ? (uint32_t)i1 + kM1 : (uint32_t)i1;
#endif
}
__device__ __forceinline__ uint32_t mrg_canon2(double p2) {
#if PRNGD_MRG_FLOOR
    const uint32_t c2 = __double2uint_rz(p2);
    return min(c2, c2 - kM2);  // m2 -> 0; below m2, c2 - m2 wraps above c2
#else
    const int32_t i2 = __double2int_rz(p2);
    return i2 < 0 ? (uint32_t)i2 + kM2 : (uint32_t)i2;
#endif
}
__device__ __forceinline__ uint32_t mrg_combined_b_m1(double p1, double p2) {
    return mrg_combine_m1(mrg_canon1(p1), mrg_canon2(p2));
}

// R23: uniform width-bit value: discard u with u - 1 >= T = floor(m1 / 2^width) * 2^width.
__device__ __forceinline__ uint32_t mrg_reduced(Mrg32k3a &m, uint32_t T, uint32_t mask) {
    uint32_t u;
    do {
        u = mrg_next(m) - 1u;
    } while (u >= T);
    return u & mask;
}

// R22: stream s starts from SplitMix64 outputs #3s, #3s+1, #3s+2 (six 32-bit words).
__device__ __forceinline__ Mrg32k3a mrg_stream_start(uint64_t seed, uint64_t s) {
    uint32_t wd[6];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const uint64_t o = splitmix_finalize(seed + (3 * s + i + 1) * kGamma);
        wd[2 * i] = (uint32_t)o;
        wd[2 * i + 1] = (uint32_t)(o >> 32);
    }
    Mrg32k3a m;
    m.s0 = wd[0] >= kM1 ? wd[0] - kM1 : wd[0];
    m.s1 = wd[1] >= kM1 ? wd[1] - kM1 : wd[1];
    m.s2 = wd[2] >= kM1 ? wd[2] - kM1 : wd[2];
    m.t0 = wd[3] >= kM2 ? wd[3] - kM2 : wd[3];
    m.t1 = wd[4] >= kM2 ? wd[4] - kM2 : wd[4];
    m.t2 = wd[5] >= kM2 ? wd[5] - kM2 : wd[5];
    if ((m.s0 | m.s1 | m.s2) == 0u) m.s0 = 1u;
    if ((m.t0 | m.t1 | m.t2) == 0u) m.t0 = 1u;
    return m;
}

// ---- S2: base draw, Marsaglia xor128 (Alg. 1 "r <- PRNG()") ---------------------
__device__ __forceinline__ uint32_t draw(Xs128 &s) {
    const uint32_t t = s.x ^ (s.x << 11);
    s.x = s.y;
    s.y = s.z;
    s.z = s.w;
    s.w = s.w ^ (s.w >> 19) ^ t ^ (t >> 8);
    return s.w;
}

// ---- S3: accept-reject (R3): a0 < x1 < a  <=>  (x1 - (a0+1)) < (a - a0 - 1) unsigned --
__device__ __forceinline__ bool accepted(uint32_t x1, uint32_t lo, uint32_t span) {
    return (uint32_t)(x1 - lo) < span;
}

// ---- S4 + S5: Eq.(1) and Eq.(4) in scaled integer units (R10) --------------------------------
// v = x1*2^w + x2 is exact in 64 bits; RN(v) = 2^w * RN(x1 + k*x2); subtracting C_s = 2^w*C and
// dividing by D_s = 2^w*D gives bit-for-bit the quotient RN(RN(z - C) / D) of Eq.(4).
template <bool IEEE_DIV, bool CLAMP>
__device__ __forceinline__ double eq4_scaled(uint64_t v, double Cs, double Ds, double y) {
    const double n = __dsub_rn(__ull2double_rn(v), Cs);
    double q;
    if (IEEE_DIV) {
        q = __ddiv_rn(n, Ds);
    } else {
        // Markstein: q0 = RN(n*y) is faithful; r = n - q0*D_s is exact in one FMA; the second
        // FMA rounds q0 + r*y to the correctly rounded quotient (y = RN(1/D_s)).
        const double q0 = __dmul_rn(n, y);
        const double r = __fma_rn(-q0, Ds, n);
        q = __fma_rn(r, y, q0);
    }
    if (CLAMP) q = fmin(q, kBelowOne);  // R11: literal Eq.(4) can round to 1.0 for w >= 27
    return q;
}

template <bool IEEE_DIV, bool CLAMP>
__device__ __forceinline__ double eq4_pair(uint32_t x1, uint32_t x2, uint32_t w, double Cs,
                                           double Ds, double y) {
    return eq4_scaled<IEEE_DIV, CLAMP>(((uint64_t)x1 << w) | (uint64_t)x2, Cs, Ds, y);
}

// ---- S5 for every mapping the library offers (runtime-uniform selection) -------------------
//   kind 4  Eq.(4):  q = RN(RN(v) - C_s) / D_s                         v = x1*2^w + x2
//   kind 5  Eq.(5):  q = RN(RN(v5) / D_s) * RN(1 - k^2)                  v5 = (x1-a0-1)*2^w + x2
//   kind 6  Eq.(6):  q = RN(RN(1 - k^2) * RN(RN(v) - 2^w)) / D_s
// each followed by the R11 clamp and, for the open interval, 1 - q.  Every 2^w
// rescaling is exact, so each is bit-identical to the literal unscaled evaluation.

template <bool IEEE_DIV, bool CLAMP>
__device__ __forceinline__ double map_pair(uint32_t x1, uint32_t x2, const MapArgs &m) {
    const uint64_t v = ((uint64_t)(x1 - m.sub) << m.w) | (uint64_t)x2;
    double n = __dsub_rn(__ull2double_rn(v), m.Cs);
    if (m.kind == 6) n = __dmul_rn(n, m.scale);
    double q;
    if (IEEE_DIV) {
        q = __ddiv_rn(n, m.Ds);
    } else {
        const double q0 = __dmul_rn(n, m.y);
        const double r = __fma_rn(-q0, m.Ds, n);
        q = __fma_rn(r, m.y, q0);
    }
    if (m.kind == 5) q = __dmul_rn(q, m.scale);
    if (CLAMP) q = fmin(q, kBelowOne);
    if (m.open) q = __dsub_rn(1.0, q);
    return q;
}

// ---- S7: bin of the 2^16-bin histogram (R16): exact scaling by 2^16, truncation -------------
__device__ __forceinline__ uint32_t bin16(double q) {
    return min((uint32_t)__double2uint_rz(__dmul_rn(q, 65536.0)), 65535u);  // R18: q = 1 (open)
}

}  // namespace prngd
