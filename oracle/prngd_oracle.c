/*
 * prngd_oracle.c -- plain, slow, obviously-correct CPU oracle.  TEST INFRASTRUCTURE ONLY
 * (see prngd_oracle.h for who may use it).  Build:
 *     gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -o liboracle_prngd.so prngd_oracle.c
 *
 * The method (§2):
 *   Eq.(1)  z = x1 + k*x2, k = 2^-w
 *   Eq.(3)  f(z) constant on [a0 + k*b ; a + k*b0]
 *   rule    "if x1=a0 or x1=a then we drop such values and take next pair"
 *   Eq.(4)  z' = (z - (a0 + k*b)) / (a - a0 - k*(b - b0))
 *   Alg. 1  PRNGD(k, min, max): draw, reject, compose, map
 * Readings of the paper where it is silent are numbered R1..R16 in DESIGN.md and cited below.
 */
#include "prngd_oracle.h"
#include <math.h>
#include <string.h>

#define GAMMA 0x9E3779B97F4A7C15ull /* SplitMix64 increment (golden ratio), R6 */

uint64_t oracle_mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t oracle_splitmix64_output(uint64_t seed, uint64_t i)
{
    /* Sequential definition: state += gamma; return mix64(state).  The (i+1)-th state is
     * seed + (i+1)*gamma mod 2^64.  Written as a loop-free product on purpose; the pin test
     * compares it with the sequential recurrence. */
    return oracle_mix64(seed + (i + 1u) * GAMMA);
}

uint32_t oracle_xs128_next(uint32_t st[4])
{
    /* Marsaglia, "Xorshift RNGs", J. Stat. Softw. 8(14), 2003, xor128. */
    uint32_t t = st[0] ^ (st[0] << 11);
    st[0] = st[1];
    st[1] = st[2];
    st[2] = st[3];
    st[3] = st[3] ^ (st[3] >> 19) ^ (t ^ (t >> 8));
    return st[3];
}

void oracle_stream_state(uint64_t seed, uint64_t s, uint32_t st[4])
{
    /* R6: global stream s takes SplitMix64 outputs #2s and #2s+1 (counter addressed). */
    uint64_t o0 = oracle_splitmix64_output(seed, 2u * s);
    uint64_t o1 = oracle_splitmix64_output(seed, 2u * s + 1u);
    st[0] = (uint32_t)(o0 & 0xFFFFFFFFu);
    st[1] = (uint32_t)(o0 >> 32);
    st[2] = (uint32_t)(o1 & 0xFFFFFFFFu);
    st[3] = (uint32_t)(o1 >> 32);
}

/* ---- NEXT-2: MRG32k3a (L'Ecuyer 1999, "Good parameters and implementations for combined
 * multiple recursive random number generators", Oper. Res. 47(1)), named by P:165. ---------- */
#define MRG_M1 4294967087ll   /* 2^32 - 209   */
#define MRG_M2 4294944443ll   /* 2^32 - 22853 */

uint32_t oracle_mrg_next(int64_t s[6])
{
    /* component 1: x_n = (1403580 x_{n-2} - 810728 x_{n-3}) mod m1 */
    int64_t p1 = (1403580ll * s[1] - 810728ll * s[0]) % MRG_M1;
    if (p1 < 0) p1 += MRG_M1;
    s[0] = s[1]; s[1] = s[2]; s[2] = p1;
    /* component 2: y_n = (527612 y_{n-1} - 1370589 y_{n-3}) mod m2 */
    int64_t p2 = (527612ll * s[5] - 1370589ll * s[3]) % MRG_M2;
    if (p2 < 0) p2 += MRG_M2;
    s[3] = s[4]; s[4] = s[5]; s[5] = p2;
    /* combination: z = (x - y) mod m1, with 0 reported as m1 -> u in [1, m1] (R21) */
    int64_t z = p1 - p2;
    if (z <= 0) z += MRG_M1;
    return (uint32_t)z;
}

void oracle_mrg_stream_state(uint64_t seed, uint64_t s, int64_t st[6])
{
    /* R22: SplitMix64 outputs #3s, #3s+1, #3s+2 -> six 32-bit words (lo, hi, ...), the first
     * three reduced mod m1, the last three mod m2; an all-zero component gets a 1. */
    uint32_t wd[6];
    for (int i = 0; i < 3; i++) {
        uint64_t o = oracle_splitmix64_output(seed, 3u * s + (uint64_t)i);
        wd[2 * i] = (uint32_t)(o & 0xFFFFFFFFu);
        wd[2 * i + 1] = (uint32_t)(o >> 32);
    }
    for (int i = 0; i < 3; i++) st[i] = (int64_t)wd[i] % MRG_M1;
    for (int i = 0; i < 3; i++) st[3 + i] = (int64_t)wd[3 + i] % MRG_M2;
    if (!st[0] && !st[1] && !st[2]) st[0] = 1;
    if (!st[3] && !st[4] && !st[5]) st[3] = 1;
}

/* R23: a uniform `width`-bit value from MRG32k3a (SPEC's reduce_to_width): with
 * T = floor(m1 / 2^width) * 2^width, draws u with u - 1 >= T are discarded, else (u-1) mod 2^width. */
uint32_t oracle_mrg_reduced(int64_t st[6], int width, uint64_t *draws)
{
    uint64_t span = 1ull << width;
    uint64_t T = ((uint64_t)MRG_M1 / span) * span;
    for (;;) {
        uint64_t u = oracle_mrg_next(st);
        (*draws)++;
        if (u - 1u < T) return (uint32_t)((u - 1u) & (span - 1u));
    }
}

static int bitlen(uint64_t v)
{
    int n = 0;
    while (v) { n++; v >>= 1; }
    return n;
}

/* R5/R13 parameter domain: 1 <= w <= 32; a < 2^32; a - a0 >= 2 (some x1 strictly inside);
 * x2 fills its draw width: b0 == 0, b + 1 a power of two, b < 2^w (so k*(b-b0) < 1). */
static int valid(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b)
{
    if (w < 1 || w > 32) return 0;
    if (a > 0xFFFFFFFFull || a0 >= a || a - a0 < 2) return 0;
    if (b0 != 0 || b == 0 || b > 0xFFFFFFFFull) return 0;
    if (((b + 1) & b) != 0) return 0;
    if (b >= (1ull << w)) return 0;
    return 1;
}

int oracle_constants(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                     double *C, double *D)
{
    if (!valid(w, a0, a, b0, b)) return 1;
    double k = ldexp(1.0, -(int)w);                       /* k = 2^-w */
    *C = (double)a0 + k * (double)b;                      /* Eq.(3) lower end a0 + k*b */
    *D = ((double)a - (double)a0) - k * ((double)b - (double)b0); /* Eq.(4) denominator */
    return 0;
}

double oracle_map_noclamp(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                          uint32_t x1, uint32_t x2)
{
    double C, D;
    if (oracle_constants(w, a0, a, b0, b, &C, &D)) return NAN;
    double k = ldexp(1.0, -(int)w);
    double t = k * (double)x2;        /* exact: power-of-two scaling              */
    double z = (double)x1 + t;        /* Eq.(1); one RN rounding when w>26 (R8) */
    double n = z - C;                 /* Eq.(4) numerator                   */
    return n / D;                     /* Eq.(4), correctly rounded division        */
}

double oracle_map(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                  uint32_t x1, uint32_t x2)
{
    double q = oracle_map_noclamp(w, a0, a, b0, b, x1, x2);
    /* R11: the literal Eq.(4) rounds to exactly 1.0 for some pairs when w >= 27; P:100 states
     * z' in [0;1), so clamp to the largest double below 1. */
    if (q >= 1.0) q = 0x1.fffffffffffffp-1;
    return q;
}

void oracle_map_array(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                      const uint32_t *x1, const uint32_t *x2, uint64_t n, int clamp, double *q)
{
    for (uint64_t i = 0; i < n; i++)
        q[i] = clamp ? oracle_map(w, a0, a, b0, b, x1[i], x2[i])
                     : oracle_map_noclamp(w, a0, a, b0, b, x1[i], x2[i]);
}

int oracle_accept(uint64_t a0, uint64_t a, uint32_t x1)
{
    /* P:95-98 drop x1 = a0 or x1 = a; R3: draws outside [a0, a] are dropped as well. */
    return (uint64_t)x1 > a0 && (uint64_t)x1 < a;
}

double oracle_map_kind(int kind, int open_interval, uint32_t w, uint64_t a0, uint64_t a,
                       uint64_t b0, uint64_t b, uint32_t x1, uint32_t x2)
{
    double q;
    if (kind == 5) q = oracle_map_eq5(w, a0, a, b0, b, x1, x2);
    else if (kind == 6) q = oracle_map_eq6(w, x1, x2);
    else q = oracle_map_noclamp(w, a0, a, b0, b, x1, x2);
    if (q >= 1.0) q = 0x1.fffffffffffffp-1;   /* R11 for every mapping */
    if (open_interval) q = 1.0 - q;           /* P:159-161 "use 1-z instead of z" */
    return q;
}

int oracle_generate_ex(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                       uint64_t seed, uint64_t stream_begin, uint64_t n_streams,
                       uint64_t n_per_stream, int kind, int alg1, int open_interval,
                       double *out, uint32_t *pidx, uint64_t *consumed,
                       int64_t *hist, double *pw, int64_t *count)
{
    return oracle_generate_gen(w, a0, a, b0, b, seed, stream_begin, n_streams, n_per_stream, kind,
                               alg1, open_interval, 0, out, pidx, consumed, hist, pw, count);
}

int oracle_generate_gen(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                        uint64_t seed, uint64_t stream_begin, uint64_t n_streams,
                        uint64_t n_per_stream, int kind, int alg1, int open_interval, int mrg,
                        double *out, uint32_t *pidx, uint64_t *consumed,
                        int64_t *hist, double *pw, int64_t *count)
{
    if (!valid(w, a0, a, b0, b)) return 1;
    if (mrg && (bitlen(a) > 31 || bitlen(b) > 31)) return 1;
    if (kind != 4 && kind != 5 && kind != 6) return 1;
    if (kind == 6 && !(a0 == 0 && b0 == 0 && a == (1ull << w) - 1 && b == a)) return 1;
    int sh1 = 32 - bitlen(a); /* R4: x = top bits of the 32-bit draw */
    int sh2 = 32 - bitlen(b);
    for (uint64_t i = 0; i < n_streams; i++) {
        uint32_t st[4];
        int64_t ms[6];
        uint64_t mdraws = 0; /* MRG32k3a outputs consumed (NEXT-2) */
        if (mrg) oracle_mrg_stream_state(seed, stream_begin + i, ms);
        else oracle_stream_state(seed, stream_begin + i, st);
        uint64_t p = 0; /* pairs (R2) or draws (Alg. 1) consumed so far */
        for (uint64_t j = 0; j < n_per_stream; j++) {
            uint32_t x1, x2;
            if (mrg && alg1) {
                /* Alg. 1 over reduced MRG32k3a values (R23): redraw R1 alone until
                   accepted, then draw R2 */
                do {
                    x1 = oracle_mrg_reduced(ms, bitlen(a), &mdraws);
                    p++;
                } while (!oracle_accept(a0, a, x1));
                x2 = oracle_mrg_reduced(ms, bitlen(b), &mdraws);
                p++;
            } else if (mrg) {
                /* pair-drop (R2) over pairs of reduced MRG32k3a values (R23) */
                do {
                    x1 = oracle_mrg_reduced(ms, bitlen(a), &mdraws);
                    x2 = oracle_mrg_reduced(ms, bitlen(b), &mdraws);
                    p++;
                } while (!oracle_accept(a0, a, x1));
            } else if (alg1) {
                /* NEXT-2, Alg. 1: redraw R1 alone until accepted, then draw R2 */
                do {
                    x1 = oracle_xs128_next(st) >> sh1;
                    p++;
                } while (!oracle_accept(a0, a, x1));
                x2 = oracle_xs128_next(st) >> sh2;
                p++;
            } else {
                do { /* R2: pair-drop -- a rejected x1 discards its whole pair */
                    uint32_t u1 = oracle_xs128_next(st);
                    uint32_t u2 = oracle_xs128_next(st);
                    x1 = u1 >> sh1;
                    x2 = u2 >> sh2;
                    p++;
                } while (!oracle_accept(a0, a, x1));
            }
            double q = oracle_map_kind(kind, open_interval, w, a0, a, b0, b, x1, x2);
            uint64_t o = i * n_per_stream + j; /* R15: stream-major layout */
            if (out) out[o] = q;
            /* pair index (R2), or index of the accepted x1 draw (Alg. 1) */
            if (pidx) pidx[o] = (uint32_t)(alg1 ? p - 2 : p - 1);
            if (hist) {
                uint32_t bin = (uint32_t)(q * 65536.0);              /* R16 */
                if (bin > 65535u) bin = 65535u;                      /* R18: q = 1 (open) */
                hist[bin]++;
            }
            if (pw) {
                double z2 = q * q;
                pw[0] += q;
                pw[1] += z2;
                pw[2] += z2 * q;
                pw[3] += z2 * z2;
            }
            if (count) (*count)++;
        }
        if (consumed) consumed[i] = mrg ? mdraws : p;
    }
    return 0;
}

int oracle_generate(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                    uint64_t seed, uint64_t stream_begin, uint64_t n_streams, uint64_t n_per_stream,
                    double *out, uint32_t *pidx, uint64_t *consumed,
                    int64_t *hist, double *pw, int64_t *count)
{
    return oracle_generate_ex(w, a0, a, b0, b, seed, stream_begin, n_streams, n_per_stream,
                              4, 0, 0, out, pidx, consumed, hist, pw, count);
}

void oracle_raw(uint64_t seed, uint64_t stream_begin, uint64_t n_streams, uint64_t draws,
                uint32_t *raw)
{
    for (uint64_t i = 0; i < n_streams; i++) {
        uint32_t st[4];
        oracle_stream_state(seed, stream_begin + i, st);
        for (uint64_t d = 0; d < draws; d++) raw[i * draws + d] = oracle_xs128_next(st);
    }
}

int oracle_enumerate(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                     double *q, uint8_t *acc)
{
    if (!valid(w, a0, a, b0, b)) return 1;
    int l1 = bitlen(a), l2 = bitlen(b);
    if (l1 + l2 > 34) return 1; /* brute force is for small widths */
    uint64_t n1 = 1ull << l1, n2 = 1ull << l2;
    for (uint64_t x1 = 0; x1 < n1; x1++)
        for (uint64_t x2 = 0; x2 < n2; x2++) {
            uint64_t o = x1 * n2 + x2;
            if (q) q[o] = oracle_map(w, a0, a, b0, b, (uint32_t)x1, (uint32_t)x2);
            if (acc) acc[o] = (uint8_t)oracle_accept(a0, a, (uint32_t)x1);
        }
    return 0;
}

double oracle_map_eq5(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                      uint32_t x1, uint32_t x2)
{
    /* Eq.(5), with grid values x = k*i (R1): trunc[(x1-a0-k)/k] = i1-a0-1 and
     * trunc[(a-a0-2k)/k] = a-a0-2 are integers; x2-b0 and b-b0 stay in units of 1 (k*i). */
    if (!valid(w, a0, a, b0, b)) return NAN;
    double k = ldexp(1.0, -(int)w);
    double kp = k * k;                                        /* k' = k^2 */
    double num = (double)((uint64_t)x1 - a0 - 1) + k * ((double)x2 - (double)b0);
    double den = (double)(a - a0 - 2) + k * ((double)b - (double)b0);
    return num / den * (1.0 - kp);
}

double oracle_map_eq6(uint32_t w, uint32_t x1, uint32_t x2)
{
    /* Eq.(6): z' = (1-k^2)(trunc[x1/k] + x2 - 1) / (trunc[1/k] - 2 - k), with the
     * grid x1 = k*i1, x2 = k*i2, so trunc[x1/k] = i1, x2 = k*i2 and trunc[1/k] = 2^w. */
    double k = ldexp(1.0, -(int)w);
    double num = (1.0 - k * k) * ((double)x1 + k * (double)x2 - 1.0);
    double den = ldexp(1.0, (int)w) - 2.0 - k;
    return num / den;
}
