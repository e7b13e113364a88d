/*
 * prngd_oracle.h -- CPU ORACLE for the PRNGD hot path (Demchik & Gulov, arXiv 1401.8230).
 *
 * TEST INFRASTRUCTURE ONLY.  This is the plain, slow, single-threaded reference that the CUDA
 * path is checked against.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load or call it.  It shares no code, header, constant table or helper
 * with paper_1401_8230_b200/ (the product), and the product never includes or links it.
 *
 * Paper citations use PAPER.md line numbers ("P:57") and equation numbers.  Every floating-point
 * operation is IEEE binary64, round-to-nearest-even, one rounding per operation, compiled with
 * -ffp-contract=off (no FMA contraction) on x86-64 SSE2.
 *
 * Parity status per function:
 *   oracle_mix64 / oracle_splitmix64_output ... pinned (published SplitMix64 seed-0 outputs)
 *   oracle_xs128_next ......................... pinned (Marsaglia 2003 xor128 example sequence)
 *   oracle_stream_state ....................... convention (R6); pinned only through the
 *                                               two primitives above + regression vectors
 *   oracle_constants / oracle_map ............. pinned (exact-rational closed form for w<=26,
 *                                               exact error bound for w>26, hand-derived constants,
 *                                               exhaustive clamp set at w=32)
 *   oracle_generate ........................... pinned (w=8 brute-force lattice, rejection rate,
 *                                               shard invariance, moments vs exact lattice moments)
 *   oracle_enumerate .......................... pinned (closed form, all 2^(2w) pairs)
 *   oracle_map_eq5 / oracle_map_eq6 ........... pinned (exact rational Eq.(5), endpoint values P:133-135)
 */
#ifndef PRNGD_ORACLE_H
#define PRNGD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64 finaliser (Steele, Lea, Flood 2014).  Seeding is not fixed by the paper (R6). */
uint64_t oracle_mix64(uint64_t z);
/* i-th output (0-based) of the SplitMix64 sequence seeded with `seed`: mix64(seed + (i+1)*gamma). */
uint64_t oracle_splitmix64_output(uint64_t seed, uint64_t i);

/* Marsaglia (2003) xor128: state (x,y,z,w) advanced in place, returns the new w.  The paper's
 * "r <- PRNG()" (Alg. 1). */
uint32_t oracle_xs128_next(uint32_t st[4]);

/* Initial xorshift128 state of global stream s (R6): outputs #2s and #2s+1 of
 * SplitMix64(seed), split into (lo32, hi32, lo32, hi32). */
void oracle_stream_state(uint64_t seed, uint64_t s, uint32_t st[4]);

/* Parameter check + Eq.(3)/(4) constants:
 *   C = a0 + k*b,  D = (a - a0) - k*(b - b0),  k = 2^-w.   Returns 0 on success, 1 if invalid. */
int oracle_constants(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                     double *C, double *D);

/* Eq.(4) for one pair (x1, x2) in integer units (R1), literal op order
 *   t = k*x2; z = x1 + t  (Eq.(1));  n = z - C;  q = n / D  (Eq.(4))
 * then the clamp q <= 1 - 2^-53 (R11).  No acceptance test here. */
double oracle_map(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                  uint32_t x1, uint32_t x2);
/* Same without the clamp (to exhibit the literal 1.0 results, R11). */
double oracle_map_noclamp(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                          uint32_t x1, uint32_t x2);

/* Element-wise oracle_map (clamp != 0) or oracle_map_noclamp over n pairs. */
void oracle_map_array(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                      const uint32_t *x1, const uint32_t *x2, uint64_t n, int clamp, double *q);

/* Accept-reject rule: accept iff a0 < x1 < a. */
int oracle_accept(uint64_t a0, uint64_t a, uint32_t x1);

/* The whole path (Alg. 1 generalised, pair-drop reading DESIGN.md R2) for global streams
 * [stream_begin, stream_begin + n_streams), n_per_stream accepted outputs each.  Every output
 * pointer may be NULL.  out/pidx: [n_streams][n_per_stream]; consumed: [n_streams];
 * hist (65536 int64), pw (4 doubles: sum q, q^2, q^3, q^4) and count are ACCUMULATED (+=).
 * Returns 0, or 1 on invalid parameters. */
int oracle_generate(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                    uint64_t seed, uint64_t stream_begin, uint64_t n_streams, uint64_t n_per_stream,
                    double *out, uint32_t *pidx, uint64_t *consumed,
                    int64_t *hist, double *pw, int64_t *count);

/* Generalised whole path: kind = 4 (Eq.(4)), 5 (Eq.(5)) or 6 (Eq.(6), P:149-157,
 * full unit-interval range only); alg1 != 0 consumes draws as Alg. 1 does (redraw x1 alone,
 * P:115-120; consumed[] then counts draws and pidx[] holds the accepted x1's draw index);
 * open_interval != 0 returns 1 - z'.  Histogram bin of q = 1.0 is 65535 (R18). */
int oracle_generate_ex(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                       uint64_t seed, uint64_t stream_begin, uint64_t n_streams,
                       uint64_t n_per_stream, int kind, int alg1, int open_interval,
                       double *out, uint32_t *pidx, uint64_t *consumed,
                       int64_t *hist, double *pw, int64_t *count);
/* NEXT-2 base generator MRG32k3a (L'Ecuyer 1999): integer output u in [1, m1] (R21),
 * per-stream state from SplitMix64 (R22), reduced uniform width-bit values (R23). */
uint32_t oracle_mrg_next(int64_t s[6]);
void oracle_mrg_stream_state(uint64_t seed, uint64_t s, int64_t st[6]);
uint32_t oracle_mrg_reduced(int64_t st[6], int width, uint64_t *draws);
/* oracle_generate_ex with a base-generator switch: mrg != 0 draws x1, x2 as reduced MRG32k3a
 * values of bitlen(a), bitlen(b) bits (both <= 31; pair-drop, or Alg. 1 with alg1 != 0);
 * consumed[] then counts MRG outputs. */
int oracle_generate_gen(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                        uint64_t seed, uint64_t stream_begin, uint64_t n_streams,
                        uint64_t n_per_stream, int kind, int alg1, int open_interval, int mrg,
                        double *out, uint32_t *pidx, uint64_t *consumed,
                        int64_t *hist, double *pw, int64_t *count);

/* One pair through mapping `kind` (4/5/6) + clamp (R11) [+ 1 - z' when open_interval]. */
double oracle_map_kind(int kind, int open_interval, uint32_t w, uint64_t a0, uint64_t a,
                       uint64_t b0, uint64_t b, uint32_t x1, uint32_t x2);

/* Raw base draws: raw[i][d] = d-th xorshift128 output of global stream stream_begin+i. */
void oracle_raw(uint64_t seed, uint64_t stream_begin, uint64_t n_streams, uint64_t draws,
                uint32_t *raw);

/* Brute force over every pair of draw values (x1 in [0,2^bitlen(a)), x2 in [0,2^bitlen(b))),
 * q[x1 * 2^bitlen(b) + x2] = oracle_map(...), acc[...] = oracle_accept(...).  Small widths only. */
int oracle_enumerate(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                     double *q, uint8_t *acc);

/* NEXT-1: Eq.(5) on the integer lattice, literal order, and Eq.(6). */
double oracle_map_eq5(uint32_t w, uint64_t a0, uint64_t a, uint64_t b0, uint64_t b,
                      uint32_t x1, uint32_t x2);
double oracle_map_eq6(uint32_t w, uint32_t x1, uint32_t x2);

#ifdef __cplusplus
}
#endif
#endif
