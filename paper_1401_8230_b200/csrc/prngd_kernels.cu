// prngd_kernels.cu -- sm_100a kernels of the PRNGD hot path.
//
// Kernels (all bit-identical to the oracle; which one a call launches: prngd_get_info):
//   gen_kernel        S1-S6, one lane per stream (the xorshift128 state in 4 registers for the
//                     whole stream), batches of kCols = 16 outputs computed speculatively (a warp
//                     vote replays a batch exactly when a lane drew a rejected x1 or the R11
//                     clamp row); store paths: ROW (default: 32 x 64-output tiles in padded shared
//                     memory, each row written as one 512-byte burst), and the A/B paths TMA, TILE,
//                     DIRECT, ROW1K
//   gen_seg_kernel    SEG: several lanes per stream via GF(2) jump-ahead, 1 KiB row segments
//   gen_segc_kernel   SEGC: column-block CTAs via jump-ahead (A/B)
//   gen_jump_kernel   NEXT-3: one warp per stream for few-stream configs
//   gen_mrg_kernel    NEXT-2: MRG32k3a base generator in exact binary64
//   consume_kernel    S1-S7: the fused 2^16-bin histogram + power sums (optimistic packed
//                     shared-memory counters) with optional ROW stores; + its exact fallback pass
//   finalize_kernel   slab reduction into the caller's (local or peer-mapped) accumulators
//   debug_*           validation hooks of include/prngd.h
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>

#include "prngd_device.cuh"
#include "prngd_internal.h"

namespace prngd {

#ifndef PRNGD_KCOLS
#define PRNGD_KCOLS 16
#endif
// outputs per lane per batch (128 B of its row); must divide every row-tile width (the fused
// consumer's is 16).  A/B on cfg3 (ROW, 200 steps): 8 -> 780-782, 16 -> 787, 32 -> 777-779.
constexpr int kCols = PRNGD_KCOLS;
constexpr int kTileBytes = 32 * kCols * 8;  // 4 KiB per warp tile
constexpr int kNBufTma = 2;                 // tiles per warp when the TMA stores them (async)

// Tiles per warp: the TMA store reads the tile asynchronously, so it gets a ring of two; the
// smem-staged st.global flush reads it synchronously and needs one; the direct path and the
// consume-only path keep the batch in registers and need none.
template <Store ST, bool WRITE>
constexpr int ring() {
    return !WRITE || ST == Store::DIRECT || ST == Store::ROW || ST == Store::ROW1K
               ? 0
               : (ST == Store::TMA ? kNBufTma : 1);
}
constexpr int kGenWarps = 4;                // warps per CTA, generate kernel (tile paths)
#ifndef PRNGD_ROW_COLS
#define PRNGD_ROW_COLS 64
#endif
constexpr int kRowCols = PRNGD_ROW_COLS;    // ROW path: outputs per row per burst (512 B)

template <Store ST>
constexpr bool is_row() { return ST == Store::ROW || ST == Store::ROW1K; }
template <Store ST>
constexpr int row_cols() { return ST == Store::ROW1K ? 2 * kRowCols : kRowCols; }
template <Store ST>
constexpr int gen_warps() { return is_row<ST>() ? 1 : kGenWarps; }
#ifndef PRNGD_ROW_PAD
#define PRNGD_ROW_PAD 1024  // ROW tile alignment (its 16-B vector stores need 16)
#endif
template <Store ST>
constexpr size_t gen_smem() {
    return is_row<ST>() ? PRNGD_ROW_PAD + (size_t)32 * (row_cols<ST>() * 8 + 16)
                        : 1024 + (size_t)kGenWarps * (ST == Store::TMA ? 2 : 1) * kTileBytes;
}
constexpr int kConsWarpsTiles = 12;         // warps per CTA, consume kernel staging tiles in smem
#ifndef PRNGD_CONS_REG_WARPS
#define PRNGD_CONS_REG_WARPS 16  // cfg5 --no-write A/B: 12 -> 754, 16 -> 796, 20 -> 789, 24 -> 761, 28 -> 758, 32 -> 748
#endif
constexpr int kConsWarpsRegs = PRNGD_CONS_REG_WARPS;  // warps per CTA, consume kernel without tiles

// consume + ROW store: 12 warps x 4 KiB tiles (128-byte row bursts) + the 128 KiB histogram.
// A/B on cfg5 (write + histogram + moments), first kernel: 6 x 16 KiB -> 415, 8 x 8 KiB -> 526,
// 12 x 8 KiB -> 544, 16 x 4 KiB -> 561-566, 20 x 4 KiB -> 538, 24 x 4 KiB -> 525 Gd/s; current
// kernel (4 KiB tiles): 8 -> 578, 10 -> 533-542, 12 -> 598-600, 14 -> 543-548, 16 -> 582-586,
// 18 -> 527; 10-11 warps x 8 KiB -> 529-562 (cfg4 + histogram: 12 -> 574-577, 16 -> 572).
#ifndef PRNGD_CONS_ROW_WARPS
#define PRNGD_CONS_ROW_WARPS 12
#define PRNGD_CONS_ROW_COLS 16
#endif
constexpr int kConsWarpsRow = PRNGD_CONS_ROW_WARPS;
constexpr int kConsRowCols = PRNGD_CONS_ROW_COLS;
// The row-segment consumer keeps only 2-4 rows per warp in flight, so it takes 16 warps
// (A/B, same box, cfg5 / cfg3 + statistics: 12 -> 597-606 / 608-617, 14 -> 571-574 / 581-589,
// 16 -> 611-616 / 618-649 Gd/s; the ROW-tile consumer loses with 16: 559 vs 580).  Session 2,
// cfg5 best step of 10-step runs: 16 -> 692.5-694.5, 18 (96 registers, spills) -> 636-640,
// 20 (96 registers) -> 677-678 Gd/s (profiles/s2k_consumer_warps_ab.txt)
#ifndef PRNGD_CONS_SEG_WARPS
#define PRNGD_CONS_SEG_WARPS 16
#endif
constexpr int kConsWarpsSeg = PRNGD_CONS_SEG_WARPS;

template <Store ST, bool WRITE>
constexpr int cons_warps() {
    return (WRITE && ST == Store::SEG) ? kConsWarpsSeg
           : (WRITE && ST == Store::ROW) ? kConsWarpsRow
                                       : (ring<ST, WRITE>() > 0 ? kConsWarpsTiles : kConsWarpsRegs);
}
constexpr int kHistWords = 32768;  // 65536 u16 counters in pairs (128 KiB)
constexpr int kBins = 65536;
// Per-CTA slabs in global memory hold one u32 per bin (256 KiB): the epilogues unpack their
// shared-memory fields into it.

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t smem, int col,
                                             int row) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
        "r"(smem), "r"(col), "r"(row)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void sts_v2(uint32_t addr, double a, double b) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void sts_f64(uint32_t addr, double a) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(a) : "memory");
}
__device__ __forceinline__ void lds_v2(uint32_t addr, double &a, double &b) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr) : "memory");
}
#ifndef PRNGD_STORE_HINT
#define PRNGD_STORE_HINT ".cs"  // streaming: outputs are not re-read by the kernel
#endif
__device__ __forceinline__ void stg_v2_cs(double *p, double a, double b) {
    asm volatile("st.global" PRNGD_STORE_HINT ".v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b)
                 : "memory");
}

// Byte offset of element pair `chunk` (16 bytes) of row `row` in a 32 x 16 double tile, in the
// TMA SWIZZLE_128B layout: chunk c of row r lives at chunk c ^ (r & 7).  Tiles are 1 KiB aligned.
__device__ __forceinline__ uint32_t tile_off(uint32_t row, uint32_t chunk) {
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

// ------------------------------------------------------------------------------ consumer (S7)
// RED: optimistic no-return adds (see consume_kernel); BELOW1: the mapping never returns 1.0
// (Eq.(4) closed with the R11 clamp), so the R18 top-bin guard is not needed.
// Power sums kept in kPowSplit independent partial accumulators (output i of a batch adds into
// set i % kPowSplit), so the four FP64 add chains of a batch are kPowSplit times shorter; the
// partials are added in a fixed order at the end (R16 compares sums at relative 1e-12).
#ifndef PRNGD_POW_SPLIT
#define PRNGD_POW_SPLIT 2  // cfg5 A/B (same box): 1 -> 579.5-579.6, 2 -> 584.9-586.1 Gd/s
#endif
// bin index of S7 by one round-toward-zero DADD (1) or by DMUL + F2I (0)
#ifndef PRNGD_BIN_RZ
#define PRNGD_BIN_RZ 1
#endif
constexpr int kPowSplit = PRNGD_POW_SPLIT;
template <bool RED, bool BELOW1 = false>
struct ConsumerT {
    double s1[kPowSplit], s2[kPowSplit], s3[kPowSplit], s4[kPowSplit];
    uint32_t *hist;   // shared: 32768 words; word j holds bin j (low half), bin j + 32768 (high)
    int64_t *spill;   // global: carries of the packed counters, [65536]
    bool hist_only;   // warp-uniform: the full-batch paths call add_hist (no power sums)
    __device__ __forceinline__ void init(uint32_t *h, int64_t *sp, bool ho = false) {
#pragma unroll
        for (int k = 0; k < kPowSplit; ++k) s1[k] = s2[k] = s3[k] = s4[k] = 0.0;
        hist = h;
        spill = sp;
        hist_only = ho;
    }
    __device__ __forceinline__ double sum(const double (&a)[kPowSplit]) const {
        double r = a[0];
#pragma unroll
        for (int k = 1; k < kPowSplit; ++k) r = __dadd_rn(r, a[k]);
        return r;
    }
    // R16 for one output.  A word holds L + 65536*H (mod 2^32) exactly, as a sum of commutative
    // increments.  The one thread whose atomicAdd wraps the field it increments (that field of
    // the new word is 0) records the carry in `spill`, which the finalize kernel adds back:
    //   low field wrapped:  L gains 65536, the carry went into H (H -1), and if H was 0xFFFF the
    //                       word wrapped too (H +65536);   high field wrapped: H gains 65536.
    __device__ __forceinline__ void add(double q, int i = 0) {
        // power sums: the FMAs round once per term (compared at relative 1e-12, R16)
        const int k = i % kPowSplit;
        const double z2 = __dmul_rn(q, q);
        s1[k] = __dadd_rn(s1[k], q);
        s2[k] = __dadd_rn(s2[k], z2);
        s3[k] = __fma_rn(z2, q, s3[k]);
        s4[k] = __fma_rn(z2, z2, s4[k]);
        add_hist(q);
    }
    // The histogram half of R16 alone (histogram-only calls; the power sums such a call still
    // accumulates on its slow paths are never read).
    __device__ __forceinline__ void add_hist(double q) {
        // t = floor(q * 2^18) = 4 bin + 2 fraction bits (the scaling is exact, so t >> 2 is R16's
        // floor(q * 2^16)): the word's byte offset is t & 0x1FFFC and the half is bit 17, with
        // no shifts (bins b and b + 32768 share word b)
        // One DADD instead of DMUL + F2I: r = q + 2^34 rounded toward zero has ulp 2^-18 on
        // [2^34, 2^35), so for 0 <= q <= 1 its mantissa is exactly floor(q * 2^18) (<= 2^18)
        // and that is the low word of r's bit pattern -- the same t as trunc(q * 2^18).
#if PRNGD_BIN_RZ
        const uint32_t t0 = (uint32_t)__double2loint(__dadd_rz(q, 17179869184.0));
#else
        const uint32_t t0 = (uint32_t)__double2uint_rz(__dmul_rn(q, 262144.0));
#endif
        const uint32_t t = BELOW1 ? t0 : min(t0, 262143u);  // R18: q = 1 -> top bin
        const uint32_t off = t & 0x1FFFCu;
        const bool high = t >= 0x20000u;
        const uint32_t inc = (t >> 17) * 0xFFFFu + 1u;  // 1 (low field) or 0x10000 (high)
        if (RED) {
            // optimistic: no return value, no carry check; a wrapped field is detected after
            // the kernel (field sum != outputs counted) and the exact pass redoes the histogram
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_u32(hist) + off), "r"(inc)
                         : "memory");
        } else {
            const uint32_t nw = atomicAdd(&hist[off >> 2], inc) + inc;
            if (__builtin_expect(((high ? nw >> 16 : nw) & 0xFFFFu) == 0u, 0))
                carry(off >> 2, high, nw);
        }
    }
    __device__ __noinline__ void carry(uint32_t word, bool high, uint32_t nw) {
        unsigned long long *sp = reinterpret_cast<unsigned long long *>(spill);
        atomicAdd(&sp[word + (high ? 32768u : 0u)], 65536ull);
        if (!high) {
            atomicAdd(&sp[word + 32768u], 0xFFFFFFFFFFFFFFFFull);  // -1: the carry went into H
            if (nw == 0u) atomicAdd(&sp[word + 32768u], 65536ull);  // ... and wrapped the word
        }
    }
};

using Consumer = ConsumerT<false, false>;

struct NoConsumer {
    static constexpr bool hist_only = false;
    __device__ __forceinline__ void init(uint32_t *, int64_t *) {}
    __device__ __forceinline__ void add(double, int = 0) {}
    __device__ __forceinline__ void add_hist(double) {}
};

// S7 for one full batch: histogram + power sums, or (one warp-uniform branch per batch) the
// histogram alone when the call has no power-sum accumulator.
template <class Cons, int N>
__device__ __forceinline__ void consume_batch(Cons &cons, const double (&q)[N]) {
    if (cons.hist_only) {
#pragma unroll
        for (int i = 0; i < N; ++i) cons.add_hist(q[i]);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) cons.add(q[i], i);
    }
}

// Eq.(4) of one pair on the specialised paths: MODE 2/3 compose v = x1:x2 as a register pair
// (w = 32), MODE 1 as one wide multiply-add x1 * 2^w + x2 (w <= 31).
#ifndef PRNGD_COMPOSE_HILO
#define PRNGD_COMPOSE_HILO 1
#endif
template <int MODE, bool IEEE>
__device__ __forceinline__ double eq4_mode(uint32_t x1, uint32_t x2, const GenArgs &g) {
#if PRNGD_COMPOSE_HILO
    // MODE 1: the two words of x1 2^w + x2 directly (x2 < 2^w, so the low word cannot carry):
    // a 32-bit multiply-add and a high multiply, no 64-bit addend to assemble
    const uint64_t v = (MODE == 2 || MODE == 3)
                           ? (((uint64_t)x1 << 32) | (uint64_t)x2)
                           : (((uint64_t)__umulhi(x1, g.pow2w) << 32) | (uint64_t)(x1 * g.pow2w + x2));
#else
    const uint64_t v = (MODE == 2 || MODE == 3) ? (((uint64_t)x1 << 32) | (uint64_t)x2)
                                                : (uint64_t)x1 * g.pow2w + (uint64_t)x2;
#endif
    return eq4_scaled<IEEE, false>(v, g.Cs, g.Ds, g.y);
}

// Kernel MODE >= 16: the mapping fixed at compile time (NEXT-1 on the bulk path): MODE = 16 +
// 4 K + 2 OPEN + W32, K = 0 Eq.(4) (with the open interval; the closed form is MODE 1-3),
// 1 Eq.(5), 2 Eq.(6).  The same operations, in the same order, as map_pair's runtime choice.
constexpr int kModeStatic = 16;
template <int MODE>
constexpr bool mode_static() { return MODE >= kModeStatic; }
template <int MODE, bool IEEE, bool CLAMP>
__device__ __forceinline__ double map_static(uint32_t x1, uint32_t x2, const GenArgs &g) {
    constexpr int K = (MODE - kModeStatic) >> 2;
    constexpr bool OPEN = ((MODE - kModeStatic) >> 1) & 1;
    constexpr bool W32 = (MODE - kModeStatic) & 1;
    const MapArgs &m = g.map;
    const uint32_t xs = x1 - m.sub;
    const uint64_t v = W32 ? (((uint64_t)xs << 32) | (uint64_t)x2)
                           : (uint64_t)xs * g.pow2w + (uint64_t)x2;
    double n = __dsub_rn(__ull2double_rn(v), m.Cs);
    if (K == 2) n = __dmul_rn(n, m.scale);
    double q;
    if (IEEE) {
        q = __ddiv_rn(n, m.Ds);
    } else {
        const double q0 = __dmul_rn(n, m.y);
        const double r = __fma_rn(-q0, m.Ds, n);
        q = __fma_rn(r, m.y, q0);
    }
    if (K == 1) q = __dmul_rn(q, m.scale);
    if (CLAMP) q = fmin(q, kBelowOne);
    if (OPEN) q = __dsub_rn(1.0, q);
    return q;
}

// ------------------------------------------------------------------------------ one batch
// One pair of the exact path: draw until accepted, then Eq.(1)+(4) with the clamp.
template <bool EQ4, bool IEEE, bool ALG1>
__device__ __forceinline__ double exact_output(Xs128 &st, uint32_t sh1, uint32_t sh2, uint32_t w,
                                               uint32_t lo, uint32_t span, const GenArgs &g) {
    uint32_t x1, x2;
    if (ALG1) {  // NEXT-2: Alg. 1 redraws x1 alone, then draws x2
        do {
            x1 = draw(st) >> sh1;
        } while (!accepted(x1, lo, span));
        x2 = draw(st) >> sh2;
    } else {     // R2: a rejected x1 drops its whole pair
        do {
            x1 = draw(st) >> sh1;
            x2 = draw(st) >> sh2;
        } while (!accepted(x1, lo, span));
    }
    return EQ4 ? eq4_pair<IEEE, true>(x1, x2, w, g.Cs, g.Ds, g.y) : map_pair<IEEE, true>(x1, x2, g.map);
}

// kCols consecutive outputs of this lane's stream, into registers q[0..kCols).
template <int MODE, bool SPEC, bool IEEE, bool ALG1>
__device__ __forceinline__ void produce_batch(Xs128 &st, double (&q)[kCols], const GenArgs &g) {
    // MODE 2: w = 32 full range, Eq.(4) closed (every constant compiled in); MODE 3: Eq.(4),
    // w = 32 and 32-bit x1 draws (v = x1:x2 is a register pair), runtime x2 width and accept
    // band (cfg4); MODE 1: Eq.(4) with runtime ranges; MODE 0: any mapping (runtime-uniform).
    constexpr bool FULL32 = MODE == 2;
    constexpr bool EQ4 = MODE >= 1 && MODE <= 3;
    const uint32_t sh1 = (MODE == 2 || MODE == 3) ? 0u : g.sh1;
    const uint32_t sh2 = FULL32 ? 0u : g.sh2;
    const uint32_t w = (MODE == 2 || MODE == 3) ? 32u : g.w;
    const uint32_t lo = FULL32 ? 1u : g.lo;
    const uint32_t span = FULL32 ? 0xFFFFFFFEu : g.span;
    if (SPEC) {
        // Fast-path band: x1 = a - 1 is the only row whose pairs can round to 1.0 (R11, monotone
        // map), so when the clamp is needed that row goes to the exact path with the rejections.
        const uint32_t span_fast = FULL32 ? 0xFFFFFFFDu : g.span_fast;
        // Speculative: compute the batch as if every x1 were accepted and below a - 1; one warp
        // vote at the end decides whether the exact path (reject loop + clamp) redoes it.
        const Xs128 saved = st;
        bool rej = false;
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
            const uint32_t x1 = draw(st) >> sh1;
            const uint32_t x2 = draw(st) >> sh2;
            rej |= !accepted(x1, lo, span_fast);
            q[i] = EQ4 ? eq4_mode<MODE, IEEE>(x1, x2, g)
                       : mode_static<MODE>() ? map_static<MODE, IEEE, false>(x1, x2, g)
                                             : map_pair<IEEE, false>(x1, x2, g.map);
        }
        if (__builtin_expect(!__any_sync(0xFFFFFFFFu, rej), 1)) return;
        st = saved;
    }
#pragma unroll
    for (int i = 0; i < kCols; ++i) q[i] = exact_output<EQ4, IEEE, ALG1>(st, sh1, sh2, w, lo, span, g);
}

__device__ __forceinline__ void stg_v4_cs(double *p, double a, double b, double c, double d) {
    // one full 32-byte sector per lane (sm_100 256-bit store)
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
                 "d"(d)
                 : "memory");
}

// Warp-coalesced flush of a 32 x 16 tile.  VEC16: 8 lanes per 128-byte row, 4 rows per
// instruction (needs a 16-byte aligned output and even nps); else 16 lanes x 8 bytes per row.
template <bool VEC16>
__device__ __forceinline__ void flush_stg(uint32_t tile, uint32_t lane, const GenArgs &g,
                                          uint64_t row0, uint64_t col0) {
    if (VEC16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t r = k * 4 + (lane >> 3), c = lane & 7u;
            double a, b;
            lds_v2(tile + tile_off(r, c), a, b);
            const uint64_t row = row0 + r, col = col0 + 2 * c;
            if (row < g.n_streams && col < g.nps) stg_v2_cs(g.out + row * g.nps + col, a, b);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t r = k * 2 + (lane >> 4), e = lane & 15u;
            double a, b;
            lds_v2(tile + tile_off(r, e >> 1), a, b);
            const uint64_t row = row0 + r, col = col0 + e;
            if (row < g.n_streams && col < g.nps) g.out[row * g.nps + col] = (e & 1u) ? b : a;
        }
    }
}

// One warp-task: streams [row0, row0 + 32), all nps columns.  `it` counts batches issued by
// this warp (tile ring position).
template <int MODE, bool SPEC, bool IEEE, bool ALG1, Store ST, bool WRITE, bool CONSUME,
          int NB, class Cons>
__device__ __forceinline__ void run_rows(const CUtensorMap *tmap, const GenArgs &g,
                                         uint32_t tiles, uint32_t lane, uint64_t row0,
                                         Cons &cons, uint32_t &it) {
    Xs128 st = stream_start(g.seed, g.stream_begin + row0 + lane);
    const bool live = (row0 + lane) < g.n_streams;  // ragged last warp: extra lanes not counted
    double *row_out = (WRITE && ST == Store::DIRECT) ? g.out + (row0 + lane) * g.nps : nullptr;
#pragma unroll 1
    for (uint64_t col0 = 0; col0 < g.nps; col0 += kCols, ++it) {
        double q[kCols];
        produce_batch<MODE, SPEC, IEEE, ALG1>(st, q, g);
        // Outputs past nps in the last batch are computed but neither stored nor counted.
        const bool full = g.nps - col0 >= (uint64_t)kCols;
        const uint32_t valid = full ? (uint32_t)kCols : (uint32_t)(g.nps - col0);
        if (CONSUME && live) {
            if (full) {
                consume_batch(cons, q);
            } else {
#pragma unroll
                for (int i = 0; i < kCols; ++i)
                    if ((uint32_t)i < valid) cons.add(q[i], i);
            }
        }
        if constexpr (!WRITE) continue;
        if constexpr (ST == Store::DIRECT) {
            // Each lane writes its own row: 4 x 32-byte full-sector stores per batch.
            if (live) {
                if (full) {
#pragma unroll
                    for (int i = 0; i < kCols; i += 4)
                        stg_v4_cs(row_out + col0 + i, q[i], q[i + 1], q[i + 2], q[i + 3]);
                } else {
#pragma unroll
                    for (int i = 0; i < kCols; ++i)
                        if ((uint32_t)i < valid) row_out[col0 + i] = q[i];
                }
            }
        } else {
        const uint32_t tile = tiles + (NB <= 1 ? 0u : (it % NB) * kTileBytes);
        if constexpr (ST == Store::TMA) {
            if (lane == 0) bulk_wait_read<NB - 1>();  // this tile's previous store read smem
            __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < kCols / 2; ++c) sts_v2(tile + tile_off(lane, c), q[2 * c], q[2 * c + 1]);
        if constexpr (ST == Store::TMA) {
            fence_proxy_async_smem();  // st.shared -> visible to the TMA (async proxy)
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(tmap, tile, (int)col0, (int)row0);
                bulk_commit();
            }
        } else {
            __syncwarp();
            flush_stg<ST == Store::STG16>(tile, lane, g, row0, col0);
            __syncwarp();  // tile reads done before the ring comes back to it
        }
        }
    }
}

// ROW store path: the warp stages kRowCols outputs of each of its 32 rows in a 16 KiB tile
// (row r, 16-byte chunk c stored at chunk c ^ r: conflict-free both for the per-lane writes and
// for the per-row reads), then writes every row as ONE 512-byte burst: 32 lanes x 16 bytes of
// the same row per st.global.  Long per-row bursts are what keeps HBM writes efficient with
// 2^20 independent row fronts (tools/pattern_sweep.py).
// Batch producers: kCols consecutive outputs of one stream into registers.
template <int MODE, bool SPEC, bool IEEE, bool ALG1>
struct XsProducer {  // xorshift128 base generator (S1-S5)
    Xs128 st;
    __device__ __forceinline__ XsProducer(const GenArgs &g, uint64_t s)
        : st(stream_start(g.seed, s)) {}
    __device__ __forceinline__ void operator()(double (&q)[kCols], const GenArgs &g) {
        produce_batch<MODE, SPEC, IEEE, ALG1>(st, q, g);
    }
};

// MRG32k3a without divergent draw loops.  A lane turns every draw into predicated logic: the
// R23 reduce-to-width test, then the value is appended to a per-lane ring of valid draws in
// shared memory (x1 at even, x2 at odd positions of the valid sequence); a valid x2 whose x1
// lies outside the band retracts the pair (pair-drop), so the ring only ever holds
// accepted pairs plus at most one pending x1.  The warp draws 3 values per lane per step (the
// unroll by the MRG's period-3 register rotation, so the state needs no moves) until every lane
// holds a batch; lanes ahead keep drawing while their ring has room, which evens out the
// per-lane acceptance luck across batches.  The consumption order of every stream is exactly
// the sequential one (NEXT-2).
#ifndef PRNGD_MRG_RING
#define PRNGD_MRG_RING 32
#endif
constexpr uint32_t kMrgRing = PRNGD_MRG_RING;      // pairs per lane (power of two, >= kCols)
constexpr uint32_t kMrgRingBytes = kMrgRing * 8u;  // per lane: 2 kMrgRing 4-byte draws
// Output staging of the MRG kernel: 0 = a ROW tile beside the rings; 1 = register stores, no
// tile (A/B: 283 vs 304 Gd/s); 2 = staged in the ring bytes the batch just consumed (no tile,
// 25 instead of 17 warps per SM; bit-exact, A/B: 324.5 vs 330.5 Gd/s -- not occupancy-bound)
#ifndef PRNGD_MRG_STAGE
#define PRNGD_MRG_STAGE 0
#endif
#ifndef PRNGD_MRG_STEP
// draws per lane per fill-loop step of the generate kernel (a multiple of the period 3); round 1
// A/B on mrg26: 3 -> 304, 6 -> 326, 9 -> 330, 12-18 -> 328-331, 24 -> 313 Gd/s; after the round-2
// cuts 15 is best (table below)
#define PRNGD_MRG_STEP 15
#endif
constexpr uint32_t kMrgStep = PRNGD_MRG_STEP;
// the fused consumer's fill step (its own optimum: A/B after the round-2 cuts, mrg26, same box,
// two alternating repetitions, write / write + statistics / statistics only in Gd/s:
//   step 9: 394.4 / 305.4 / 332.7;  12: 395.7 / 310.6 / -;  15: 400.0 / 316.2 / 344.2;
//   18: 397.4 / 318.1 / 342.0;  21: 389.5 / 309.6 / 337.7;  24: 379.0 / 304.8 / 328.2;
//   30: 351.2 / 282.2 / 301.7 -- profiles/s2j_mrg_step_ab.txt)
#ifndef PRNGD_MRG_STEP_CONS
#define PRNGD_MRG_STEP_CONS 18
#endif
constexpr uint32_t kMrgStepCons = PRNGD_MRG_STEP_CONS;
static_assert(kMrgStep % 3 == 0 && kMrgStepCons % 3 == 0, "the register rotation has period 3");
// a lane one draw short of a batch must still have room for a whole step (else the fill loop
// never ends)
static_assert(kMrgRingBytes >= 8u * kCols + 4u * (kMrgStep > kMrgStepCons ? kMrgStep : kMrgStepCons),
              "MRG ring smaller than batch + step");

// MRG_FP64: 0 = both components in 32-bit integer arithmetic, 1 = component 1 in binary64,
// 2 = both in binary64 (exact either way; A/B of INT32 vs FP64 pipe load)
#ifndef PRNGD_MRG_FP64
#define PRNGD_MRG_FP64 2
#endif
// REGCONST: the moduli and reciprocals pinned in registers for the generate kernel (A/B on
// mrg26, same box, two alternating repetitions: write 387.6 -> 394.6 Gd/s; the fused consumer,
// short of registers, 301.0 -> 299.4, so it keeps the constant-bank operands)
#ifndef PRNGD_MRG_REGCONST
#define PRNGD_MRG_REGCONST 1
#endif
#ifndef PRNGD_MRG_REGCONST_CONS
#define PRNGD_MRG_REGCONST_CONS 0  // the same for the fused consumer (A/B only: at fill step 18
                                   // 316.8 vs 318.3 Gd/s write + statistics, 341.4 vs 342.0 stats only)
#endif
template <int FP> struct MrgWord { using T = uint32_t; };
template <> struct MrgWord<1> { using T = double; };
// SPECB slow path: rewrite a lane's buffered draws [rd, wr) of its ring (counter c at shared
// address (c & (kMrgRingBytes - 4)) ^ ring, `ring` = MrgProducer2::cx) without the out-of-band x1 (and, pair-drop, its x2), in order; a trailing pending x1
// stays pending (pair-drop drops its pair once the x2 is drawn).  Returns the new write counter.
template <bool ALG1>
__device__ __noinline__ uint32_t mrg_drop_out_of_band(uint32_t ring, uint32_t rd, uint32_t wr,
                                                      uint32_t lo, uint32_t span) {
    uint32_t src = rd, dst = rd;
    bool expect_x1 = true;
    while (src != wr) {
        uint32_t x;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"((src & (kMrgRingBytes - 4u)) ^ ring));
        bool keep = true;
        if (expect_x1 && !accepted(x, lo, span)) {
            if (ALG1) {
                keep = false;             // Alg. 1: redraw x1 alone
            } else if (src + 4u != wr) {
                keep = false;             // pair-drop: the x2 goes with it
                src += 4u;
            }                             // else pending: kept, dropped once its pair completes
        }
        if (keep) {
            asm volatile("st.shared.u32 [%0], %1;" ::"r"((dst & (kMrgRingBytes - 4u)) ^ ring), "r"(x)
                         : "memory");
            dst += 4u;
            expect_x1 = !expect_x1;
        }
        src += 4u;
    }
    return dst;
}

// SPECB: the band test is taken out of the per-draw path (the host chose it because fewer than
// 1 in 4096 x1 fall outside the band): every valid draw is appended, a batch checks its 16 x1
// when it is read, and a warp with an out-of-band x1 compacts those lanes' rings (dropping the
// pair, or the x1 alone for Alg. 1), refills and reads again.
// SWZ: the ring entries are XOR-swizzled by 16 (lane mod 16) bytes instead of the counters being
// staggered, so every batch is one ring half (counter 0 or 128 mod 256) and reads its 16 pairs
// with eight 16-byte loads at base ^ 16 c (conflict-free: lane l's chunk c sits in bank group
// c ^ (l mod 8)) instead of sixteen 8-byte loads with a wrapped address each; appends at equal
// counters meet at most two lanes per bank, as the stagger did.  A/B on mrg26: 71.4 instead of
// ~73.4 instructions per output, but 368.4 against 374.5 Gd/s (more fixed-latency "wait" stalls,
// issue 75% -> 72%; profiles/r02z_mrg_swz_ab.txt), so it stays a build knob.
#ifndef PRNGD_MRG_SWZ
#define PRNGD_MRG_SWZ 0
#endif
template <bool EQ4, bool SAMEW, bool ALG1 = false, bool SPECB = false, bool SWZ = false,
          bool RC = false, uint32_t STEP = kMrgStep>
struct MrgProducer2 {  // SAMEW: x1 and x2 have the same width (one threshold and mask)
    using T1 = typename MrgWord<PRNGD_MRG_FP64 >= 1 ? 1 : 0>::T;  // component 1 word
    using T2 = typename MrgWord<PRNGD_MRG_FP64 >= 2 ? 1 : 0>::T;  // component 2 word
    const GenArgs &k;  // moduli and reciprocals (constant bank)
    T1 A, B, C;                 // component 1, oldest..newest (rotating roles)
    T2 D, E, F;                 // component 2
    // ring byte counters (free-running, 4 per draw).  Without SWZ both start at stride * lane:
    // lane l's entries are rotated so lanes at equal counts use different banks; with SWZ both
    // start at 0 and the addresses carry the bank spread.  The ring is kMrgRingBytes aligned, so
    // an entry's address is (counter & (kMrgRingBytes - 4)) ^ cx
    uint32_t wr, rd;
    uint32_t bad1;              // 4: the pending x1 lies outside the band, else 0
    uint32_t cx;                // this lane's ring (shared address) | its SWZ swizzle
    // RC: moduli and reciprocals pinned in registers (passed through a warp shuffle, which ptxas
    // cannot rematerialise as a constant-bank load inside the fill loop: the round-down FMA's
    // immediate shift takes its one non-register operand slot)
    double m1r, i1r, m2r, i2r;
    // stride: the counters of lane l start at stride * l (8: bank spread; 16: the in-ring output
    // staging of PRNGD_MRG_STAGE = 2 and of the fused consumer)
    __device__ __forceinline__ MrgProducer2(const GenArgs &g, uint64_t s, uint32_t ring_base,
                                            uint32_t lane,
                                            uint32_t stride = PRNGD_MRG_STAGE == 2 ? 16u : 8u)
        : k(g) {
        if constexpr (RC) {
            m1r = __shfl_sync(0xFFFFFFFFu, g.mrg_m1, 0);
            i1r = __shfl_sync(0xFFFFFFFFu, g.mrg_inv1, 0);
            m2r = __shfl_sync(0xFFFFFFFFu, g.mrg_m2, 0);
            i2r = __shfl_sync(0xFFFFFFFFu, g.mrg_inv2, 0);
        }
        const Mrg32k3a m = mrg_stream_start(g.seed, s);
        A = (T1)m.s0, B = (T1)m.s1, C = (T1)m.s2, D = (T2)m.t0, E = (T2)m.t1, F = (T2)m.t2;
        rd = wr = SWZ ? 0u : stride * lane;
        bad1 = 0u;
        cx = SWZ ? (ring_base | (16u * (lane & 15u))) : ring_base;
    }
    static __device__ __forceinline__ uint32_t c1(uint32_t a, uint32_t b) { return mrg_c1(a, b); }
    __device__ __forceinline__ double c1(double a, double b) const {
        return RC ? mrg_c1d(a, b, m1r, i1r) : mrg_c1d(a, b, k.mrg_m1, k.mrg_inv1);
    }
    static __device__ __forceinline__ uint32_t c2(uint32_t a, uint32_t b) { return mrg_c2(a, b); }
    __device__ __forceinline__ double c2(double a, double b) const {
        return RC ? mrg_c2d(a, b, m2r, i2r) : mrg_c2d(a, b, k.mrg_m2, k.mrg_inv2);
    }
    // u - 1 of the combined draw (R21), the value R23 tests
    static __device__ __forceinline__ uint32_t combine(uint32_t p1, uint32_t p2) {
        return mrg_combine_m1(p1, p2);
    }
    static __device__ __forceinline__ uint32_t combine(double p1, double p2) {
        return mrg_combined_b_m1(p1, p2);
    }
    static __device__ __forceinline__ uint32_t combine(double p1, uint32_t p2) {
        return mrg_combine_m1(mrg_canon1(p1), p2);
    }
    __device__ __forceinline__ void take(uint32_t x, const GenArgs &g) {  // x = u - 1
        const uint32_t odd = wr & 4u;  // 4: this draw would be an x2
        const bool v = x < (SAMEW ? g.mrg_t1 : (odd ? g.mrg_t2 : g.mrg_t1));  // R23
        const uint32_t xm = x & (SAMEW ? g.mrg_mask1 : (odd ? g.mrg_mask2 : g.mrg_mask1));
        // entry address (wr & (kMrgRingBytes - 4)) ^ cx as ONE three-input LOP3 (ptxas splits
        // the C expression into an AND and an XOR)
        uint32_t ea;
        asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(ea) : "r"(wr), "r"(kMrgRingBytes - 4u), "r"(cx));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                     "@p st.shared.u32 [%0], %1;\n\t}" ::"r"(ea),
                     "r"(xm), "r"((uint32_t)v)
                     : "memory");
        // a valid x2 completes the pair: kept (+4) or dropped with its x1 (-4).  bad1
        // (4 = the pending x1 is outside the band) is rewritten by every valid draw; only an
        // x1's value is ever read (at the next valid draw, which is then an x2)
        if (SPECB) {  // band checked when the batch is read
            wr = v ? wr + 4u : wr;
            return;
        }
        const uint32_t bad = accepted(xm, g.lo, g.span) ? 0u : 4u;
        if (ALG1) {
            // Alg. 1: an x1 outside the band is redrawn alone (not kept), x2 is
            // never tested
            const bool keep = odd != 0u || bad == 0u;
            wr = (v && keep) ? wr + 4u : wr;
        } else {
            const uint32_t d = 4u - ((odd & bad1) << 1);
            wr = v ? wr + d : wr;
            bad1 = v ? bad : bad1;
        }
    }
    __device__ __forceinline__ void fill(const GenArgs &g) {
#pragma unroll 1
        while (__any_sync(0xFFFFFFFFu, wr - rd < 8u * (uint32_t)kCols)) {
            if (wr - rd <= kMrgRingBytes - 4u * STEP) {  // room for STEP more draws
#pragma unroll
                for (int r = 0; r < (int)STEP / 3; ++r) {
                    A = c1(B, A), D = c2(F, D);
                    take(combine(A, D), g);
                    B = c1(C, B), E = c2(D, E);
                    take(combine(B, E), g);
                    C = c1(A, C), F = c2(E, F);
                    take(combine(C, F), g);
                }
            }
        }
    }
    __device__ __forceinline__ void operator()(double (&q)[kCols], const GenArgs &g) {
        uint32_t a1[kCols], a2[kCols];
#pragma unroll 1
        while (true) {
            fill(g);
            if constexpr (SWZ) {
                static_assert(8u * kCols == kMrgRingBytes / 2, "SWZ: a batch is half a ring");
                const uint32_t bh = cx ^ (rd & (kMrgRingBytes / 2));  // this batch's half
#pragma unroll
                for (int c = 0; c < kCols / 2; ++c)
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(a1[2 * c]), "=r"(a2[2 * c]), "=r"(a1[2 * c + 1]),
                                   "=r"(a2[2 * c + 1])
                                 : "r"(bh ^ (16u * c)));
            } else {
#pragma unroll
                for (int i = 0; i < kCols; ++i)
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                                 : "=r"(a1[i]), "=r"(a2[i])
                                 : "r"(((rd + 8u * i) & (kMrgRingBytes - 8u)) ^ cx));
            }
            if (!SPECB) break;
            bool bad = false;
#pragma unroll
            for (int i = 0; i < kCols; ++i) bad |= !accepted(a1[i], g.lo, g.span);
            if (__builtin_expect(!__any_sync(0xFFFFFFFFu, bad), 1)) break;
            if (bad) wr = mrg_drop_out_of_band<ALG1>(cx, rd, wr, g.lo, g.span);
        }
#pragma unroll
        for (int i = 0; i < kCols; ++i)
            q[i] = EQ4 ? eq4_mode<1, false>(a1[i], a2[i], g) : map_pair<false, true>(a1[i], a2[i], g.map);
        if (EQ4 && g.span != g.span_fast) {  // R11 clamp only where the host found it needed
#pragma unroll
            for (int i = 0; i < kCols; ++i) q[i] = fmin(q[i], kBelowOne);
        }
        rd += 8u * kCols;
    }
};

// BULK (A/B): full tiles leave through the copy engine instead of LDS + STG: every lane issues
// one cp.async.bulk of its own 512-byte row segment (shared -> global) and waits for the copy's
// shared-memory reads before it overwrites the row.
#ifndef PRNGD_ROW_BULK
#define PRNGD_ROW_BULK 0
#endif
__device__ __forceinline__ void bulk_s2g(double *dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(src), "r"(bytes)
                 : "memory");
}
template <bool CONSUME, int RC, class Prod, class Cons, bool BULK = false>
__device__ __forceinline__ void run_rows_burst(const GenArgs &g, uint32_t tile, uint32_t lane,
                                               uint64_t row0, Prod &prod, Cons &cons) {
    constexpr uint32_t CPR = RC / 2;  // 16-byte chunks per row segment
    const bool live = (row0 + lane) < g.n_streams;
    const uint32_t nrows = (g.n_streams - row0) < 32u ? (uint32_t)(g.n_streams - row0) : 32u;
    // tile row stride RC * 8 + 16 bytes: the 16-byte pad staggers the rows over the banks, so
    // both the per-lane row writes and the per-row flush reads are conflict-free with plain
    // (immediate-offset) addresses
    constexpr uint32_t RS = RC * 8u + 16u;
    const uint32_t my_row = tile + lane * RS;
#pragma unroll 1
    for (uint64_t col0 = 0; col0 < g.nps; col0 += RC) {
#pragma unroll 1
        for (uint32_t b = 0; b < RC / kCols; ++b) {
            double q[kCols];
            prod(q, g);
            if (BULK && b == 0) bulk_wait_read<0>();  // the previous tile's copy read the row
            if (CONSUME && live) {
                const uint64_t base = col0 + b * kCols;
                if (base + kCols <= g.nps) {
                    consume_batch(cons, q);
                } else {
#pragma unroll
                    for (int i = 0; i < kCols; ++i)
                        if (base + i < g.nps) cons.add(q[i], i);
                }
            }
#pragma unroll
            for (int c = 0; c < kCols / 2; ++c) {
                const uint32_t chunk = b * (kCols / 2) + c;  // logical 16-byte chunk of the row
                sts_v2(my_row + (chunk << 4), q[2 * c], q[2 * c + 1]);
            }
        }
        if (BULK && col0 + RC <= g.nps) {
            // each lane: its own row segment, written by itself, to its own row of the output
            fence_proxy_async_smem();
            if (live) bulk_s2g(g.out + (row0 + lane) * g.nps + col0, my_row, RC * 8u);
            bulk_commit();
            continue;
        }
        __syncwarp();
        if (BULK) bulk_wait_read<0>();
        if (nrows == 32u && col0 + RC <= g.nps) {
            // full tile: unconditional stores, pointer stepped by rows (the common case)
            constexpr uint32_t RPI = CPR >= 32 ? 1u : 32u / CPR;   // rows per instruction
            constexpr uint32_t LPR = CPR >= 32 ? 32u : CPR;        // lanes per row
            const uint32_t c = lane % LPR, rsub = lane / LPR;
#pragma unroll
            for (uint32_t h = 0; h < (CPR >= 32 ? CPR / 32 : 1u); ++h) {
                const uint32_t ch = h * 32u + c;  // this lane's 16-byte chunk of the row segment
                double *dst = g.out + (row0 + rsub) * g.nps + col0 + 2 * ch;
                const uint64_t step = (uint64_t)RPI * g.nps;
                uint32_t a = tile + rsub * RS + (ch << 4);
#pragma unroll 8
                for (uint32_t r = rsub; r < 32u; r += RPI) {
                    double v0, v1;
                    lds_v2(a, v0, v1);
                    stg_v2_cs(dst, v0, v1);
                    dst += step;
                    a += RPI * RS;
                }
            }
        } else if constexpr (CPR >= 32) {
            // one row per instruction: 32 lanes x 16 B = 512 B of the same row
#pragma unroll
            for (uint32_t h = 0; h < CPR / 32; ++h) {
                const uint64_t col = col0 + 2 * (h * 32 + lane);
                if (col < g.nps) {
                    double *dst = g.out + row0 * g.nps + col;
#pragma unroll 4
                    for (uint32_t r = 0; r < nrows; ++r) {
                        double a, b2;
                        lds_v2(tile + r * RS + ((h * 32u + lane) << 4), a, b2);
                        stg_v2_cs(dst + (uint64_t)r * g.nps, a, b2);
                    }
                }
            }
        } else {
            // 32 / CPR rows per instruction, CPR lanes per row
            const uint32_t c = lane % CPR, rsub = lane / CPR;
            const uint64_t col = col0 + 2 * c;
#pragma unroll 4
            for (uint32_t r0 = 0; r0 < 32; r0 += 32 / CPR) {
                const uint32_t r = r0 + rsub;
                if (r < nrows && col < g.nps) {
                    double a, b2;
                    lds_v2(tile + r * RS + (c << 4), a, b2);
                    stg_v2_cs(g.out + (row0 + r) * g.nps + col, a, b2);
                }
            }
        }
        __syncwarp();
    }
    if (BULK) bulk_wait_all();
}

__device__ __forceinline__ uint32_t aligned_smem_base(uint8_t *raw) {
    return (smem_u32(raw) + 1023u) & ~1023u;
}

// ------------------------------------------------------------------------------ kernels
// S1-S6.  Grid: one warp per 32 streams, kGenWarps warps per CTA.
template <int MODE, bool SPEC, bool IEEE, bool ALG1, Store ST>
__global__ void __launch_bounds__(gen_warps<ST>() * 32)
    gen_kernel(const __grid_constant__ CUtensorMap tmap, const GenArgs g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t row0 = ((uint64_t)blockIdx.x * gen_warps<ST>() + warp) * 32u;
    if constexpr (is_row<ST>()) {
        NoConsumer nc;
        XsProducer<MODE, SPEC, IEEE, ALG1> prod(g, g.stream_begin + row0 + lane);
        run_rows_burst<false, row_cols<ST>(), decltype(prod), NoConsumer,
                       (PRNGD_ROW_BULK != 0 && ST == Store::ROW)>(g, (smem_u32(smem_raw) + (PRNGD_ROW_PAD - 1u)) & ~(PRNGD_ROW_PAD - 1u),
                                                                  lane, row0, prod, nc);
    } else if constexpr (ST == Store::TMA) {
        // CTA-level staging: the 4 warps fill one 128-row x 16-column slab (16 KiB, two slots)
        // and thread 0 writes it with ONE tensor store per batch.  Warps past n_streams keep
        // computing (their rows are clipped by the TMA) so every thread reaches the barrier.
        const uint32_t slab0 = aligned_smem_base(smem_raw);
        const uint32_t my_tile = slab0 + warp * kTileBytes;
        const uint64_t cta_row0 = (uint64_t)blockIdx.x * kGenWarps * 32u;
        Xs128 st = stream_start(g.seed, g.stream_begin + row0 + lane);
        uint32_t slot = 0;
#pragma unroll 1
        for (uint64_t col0 = 0; col0 < g.nps; col0 += kCols, slot ^= 1u) {
            double q[kCols];
            produce_batch<MODE, SPEC, IEEE, ALG1>(st, q, g);
            const uint32_t tile = my_tile + slot * (kGenWarps * kTileBytes);
#pragma unroll
            for (int c = 0; c < kCols / 2; ++c)
                sts_v2(tile + tile_off(lane, c), q[2 * c], q[2 * c + 1]);
            fence_proxy_async_smem();  // st.shared -> visible to the TMA (async proxy)
            // The other slot's store (previous batch) must have read its smem before the next
            // batch overwrites it; thread 0 owns the bulk groups, the barrier publishes it.
            if (threadIdx.x == 0) bulk_wait_read<0>();
            __syncthreads();
            if (threadIdx.x == 0) {
                tma_store_2d(&tmap, slab0 + slot * (kGenWarps * kTileBytes), (int)col0,
                             (int)cta_row0);
                bulk_commit();
            }
        }
        if (threadIdx.x == 0) bulk_wait_all();
    } else {
        constexpr int NB = ring<ST, true>();
        const uint32_t tiles = aligned_smem_base(smem_raw) + warp * (NB * kTileBytes);
        if (row0 >= g.n_streams) return;
        uint32_t it = 0;
        NoConsumer nc;
        run_rows<MODE, SPEC, IEEE, ALG1, ST, true, false, NB>(&tmap, g, tiles, lane, row0, nc,
                                                                it);
    }
}

// End of a consumer CTA: moments reduced (warp tree, then per-CTA in warp order: deterministic
// for a fixed grid) into g.pow_slab, the packed histogram copied to this CTA's slab, and for the
// optimistic (RED) adds the field-sum check against the outputs counted (`expect`: this
// thread's share), which raises g.overflow when a 16-bit field wrapped.
template <bool RED, int kWarps, class Cons>
__device__ __forceinline__ void consume_epilogue(const Cons &cons, const uint32_t *hist,
                                                 const GenArgs &g, unsigned long long expect) {
    __shared__ double red[kWarps][4];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    double s[4] = {cons.sum(cons.s1), cons.sum(cons.s2), cons.sum(cons.s3), cons.sum(cons.s4)};
#pragma unroll
    for (int k = 0; k < 4; ++k)
        for (int o = 16; o > 0; o >>= 1) s[k] = __dadd_rn(s[k], __shfl_xor_sync(~0u, s[k], o));
    if (lane == 0)
        for (int k = 0; k < 4; ++k) red[warp][k] = s[k];
    __syncthreads();
    if (threadIdx.x < 4) {
        double acc = 0.0;
        for (int wi = 0; wi < kWarps; ++wi) acc = __dadd_rn(acc, red[wi][threadIdx.x]);
        g.pow_slab[blockIdx.x * 4 + threadIdx.x] = acc;
    }
    // unpack word j (bins j, j + 32768) into the u32-per-bin slab
    uint4 *lo_dst = reinterpret_cast<uint4 *>(g.hist_slab + (size_t)blockIdx.x * kBins);
    uint4 *hi_dst = lo_dst + kHistWords / 4;
    const uint4 *src = reinterpret_cast<const uint4 *>(hist);
    unsigned long long fsum = 0;  // sum of this thread's 16-bit fields (RED check)
    for (uint32_t i = threadIdx.x; i < kHistWords / 4; i += blockDim.x) {
        const uint4 v = src[i];
        const uint4 lo = make_uint4(v.x & 0xFFFFu, v.y & 0xFFFFu, v.z & 0xFFFFu, v.w & 0xFFFFu);
        const uint4 hi = make_uint4(v.x >> 16, v.y >> 16, v.z >> 16, v.w >> 16);
        lo_dst[i] = lo;
        hi_dst[i] = hi;
        if (RED) fsum += lo.x + lo.y + lo.z + lo.w + hi.x + hi.y + hi.z + hi.w;
    }
    if (RED) {
        for (int o = 16; o > 0; o >>= 1) {
            fsum += __shfl_xor_sync(~0u, fsum, o);
            expect += __shfl_xor_sync(~0u, expect, o);
        }
        __shared__ unsigned long long part[2][kWarps];
        if (lane == 0) {
            part[0][warp] = fsum;
            part[1][warp] = expect;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long a = 0, b = 0;
            for (int wi = 0; wi < kWarps; ++wi) {
                a += part[0][wi];
                b += part[1][wi];
            }
            if (a != b) atomicOr(g.overflow, 1u);
        }
    }
}

// S7 over values already in device memory (the MRG32k3a path: generate, then this kernel on
// the written outputs).  Persistent, one CTA per SM, grid-stride coalesced loads; the same
// packed histogram, optimistic adds, exact pass and slabs as consume_kernel.
constexpr int kHistMemWarps = 16;
template <bool RED, bool EXACT_GUARD>
__global__ void __launch_bounds__(kHistMemWarps * 32, 1)
    hist_mem_kernel(const double *__restrict__ src, uint64_t n, const __grid_constant__ GenArgs g) {
    if (EXACT_GUARD && *(volatile const uint32_t *)g.overflow == 0u) return;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = aligned_smem_base(smem_raw);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem_raw + (base - smem_u32(smem_raw)));
    for (uint32_t i = threadIdx.x; i < kHistWords; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    ConsumerT<RED, false> cons;
    cons.init(hist, g.hist_spill);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long counted = 0;
#pragma unroll 1
    for (; i + 3 * stride < n; i += 4 * stride) {
        double q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = __ldcs(src + i + k * stride);
#pragma unroll
        for (int k = 0; k < 4; ++k) cons.add(q[k], k);
        counted += 4;
    }
#pragma unroll 1
    for (; i < n; i += stride) {
        cons.add(__ldcs(src + i));
        ++counted;
    }
    consume_epilogue<RED, kHistMemWarps>(cons, hist, g, counted);
}

// S1-S7, persistent: one CTA per SM owning a 128 KiB packed histogram; warps take 32-stream
// tasks round-robin.  Writes per-CTA slabs that finalize_kernel reduces.
// RED: optimistic no-return shared-memory adds; the CTA then checks that its 16-bit fields sum
// to the number of outputs it counted (any wrapped field makes the sum short) and raises
// g.overflow.  EXACT_GUARD: the exact (carry-tracking) kernel of the fallback pass, which
// returns at once unless that flag is set and then rewrites every slab.
// one warp-task of the row-segment consumer (defined with the SEG kernel below)
template <int MODE, class Cons>
__device__ __forceinline__ void run_task_seg_consume(const GenArgs &g, uint32_t tile,
                                                     uint32_t lane, uint64_t t, Cons &cons);

template <int MODE, bool SPEC, bool IEEE, bool ALG1, Store ST, bool WRITE, bool RED = false,
          bool EXACT_GUARD = false>
__global__ void __launch_bounds__(cons_warps<ST, WRITE>() * 32, 1)
    consume_kernel(const __grid_constant__ CUtensorMap tmap, const GenArgs g) {
    if (EXACT_GUARD && *(volatile const uint32_t *)g.overflow == 0u) return;
    constexpr int kWarps = cons_warps<ST, WRITE>();
    constexpr int NB = ring<ST, WRITE>();
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = aligned_smem_base(smem_raw);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem_raw + (base - smem_u32(smem_raw)));
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t tiles = base + kHistWords * 4u + warp * (NB * kTileBytes);
    for (uint32_t i = threadIdx.x; i < kHistWords; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    ConsumerT<RED, (MODE >= 1 && MODE <= 3)> cons;
    cons.init(hist, g.hist_spill, g.hist_only != 0u);
    uint32_t it = 0;
    // rows per warp-task: 32, or 32 / S with S lanes per row (SEG)
    constexpr bool kSeg = WRITE && ST == Store::SEG;
    const uint32_t rpw = kSeg ? (32u >> g.seg_log2) : 32u;
    const uint64_t n_tasks = (g.n_streams + rpw - 1u) / rpw;
#pragma unroll 1
    // task t = blockIdx.x + gridDim.x * (warp + kWarps * k): the tasks in flight at any time
    // are one contiguous block (as with CTA-major order), and a small config's few tasks land
    // on different SMs instead of filling the first CTA's warps
    for (uint64_t t = (uint64_t)blockIdx.x + (uint64_t)gridDim.x * warp; t < n_tasks;
         t += (uint64_t)gridDim.x * kWarps) {
        if constexpr (WRITE && ST == Store::ROW) {
            XsProducer<MODE, SPEC, IEEE, ALG1> prod(g, g.stream_begin + t * 32u + lane);
            run_rows_burst<true, kConsRowCols>(
                g, base + kHistWords * 4u + warp * (32u * (kConsRowCols * 8u + 16u)), lane, t * 32u, prod,
                cons);
        } else if constexpr (kSeg) {
            run_task_seg_consume<MODE>(
                g, base + kHistWords * 4u + warp * (32u * (kConsRowCols * 8u + 16u)), lane, t, cons);
        } else
            run_rows<MODE, SPEC, IEEE, ALG1, ST, WRITE, true, NB>(&tmap, g, tiles, lane, t * 32u,
                                                                     cons, it);
    }
    if constexpr (WRITE && ST == Store::TMA) {
        if (lane == 0) bulk_wait_all();
    }
    // outputs this CTA counted (RED check): live rows of its tasks x nps, summed on lane 0
    unsigned long long expect = 0;
    if (RED && lane == 0)
        for (uint64_t t = (uint64_t)blockIdx.x + (uint64_t)gridDim.x * warp; t < n_tasks;
             t += (uint64_t)gridDim.x * kWarps) {
            const uint64_t left = g.n_streams - t * rpw;
            expect += (left < rpw ? left : rpw) * g.nps;
        }
    consume_epilogue<RED, kWarps>(cons, hist, g, expect);
}

// Reduce the per-CTA slabs into the caller's accumulators; resets the spill array to zero.
// The accumulators may live on another GPU (peer memory, prngd_ipc_open), so every add is a
// system-scope atomic.  With `arrive` != null the call then signals completion: each thread
// fences its adds at system scope, the last block to finish (counter `done`, in the scratch,
// reset by that block) bumps *arrive with a system-scope release -- so a reader that acquires
// *arrive >= target (prngd_wait_arrivals) sees every add of those calls.
// MC (NEXT-4): the accumulators are an NVLS multicast address (prngd_mc_bind_map): every add is
// a multimem.red, which the NVSwitch performs on every member GPU's copy (an all-reduce inside
// this kernel), and the arrival increment a multimem.red with release semantics.
template <bool MC>
__device__ __forceinline__ void stat_add_u64(unsigned long long *p, unsigned long long v) {
    if (MC)
        asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else
        atomicAdd_system(p, v);
}
template <bool MC>
__device__ __forceinline__ void stat_add_f64(double *p, double v) {
    if (MC)
        asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
    else
        atomicAdd_system(p, v);
}
template <bool MC>
__device__ __forceinline__ void red_release_sys_u64(unsigned long long *p, unsigned long long v) {
    if (MC)
        asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else
        asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
#ifndef PRNGD_FINALIZE_SPLIT
#define PRNGD_FINALIZE_SPLIT 4
#endif
constexpr uint32_t kFinalizeSplit = PRNGD_FINALIZE_SPLIT;  // slab groups per bin (1, 2, 4 or 8)
static_assert(256 % kFinalizeSplit == 0 && kBins % (256 / kFinalizeSplit) == 0, "finalize split");
template <bool MC>
__global__ void __launch_bounds__(256) finalize_kernel(const uint32_t *slab, int n_slabs,
                                                       int64_t *spill, const double *pow_slab,
                                                       int64_t *d_hist, double *d_pow,
                                                       int64_t *d_count, uint32_t *overflow,
                                                       uint32_t *done, unsigned long long *arrive) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *overflow = 0u;  // read by the exact pass before
    __shared__ long long part[8];
    __shared__ unsigned long long qsum[kFinalizeSplit][256 / kFinalizeSplit];
    long long local = 0;
    // A block owns 256 / kFinalizeSplit consecutive bins; thread t sums slab group t / (256 /
    // kFinalizeSplit) of bin t % (256 / kFinalizeSplit) with eight slabs in flight (independent
    // partial sums), so a warp reads 128 contiguous bytes per slab and ~440 requests are in flight
    // per SM: the ~39 MB of slabs of a 148-CTA consumer stream at memory speed (the first version,
    // 32 blocks striding over the bins with one serial chain per bin, took ~0.1 ms per call).
    constexpr uint32_t BPB = 256u / kFinalizeSplit;  // bins per block
    const uint32_t lb = threadIdx.x % BPB, grp = threadIdx.x / BPB;
    const uint32_t b = blockIdx.x * BPB + lb;
    const int s0 = (int)(((uint32_t)n_slabs * grp) / kFinalizeSplit);
    const int s1 = (int)(((uint32_t)n_slabs * (grp + 1)) / kFinalizeSplit);
    {
        const uint32_t *p = slab + b;
        unsigned long long a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int s = s0;
        for (; s + 8 <= s1; s += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] += p[(size_t)(s + k) * kBins];
        }
        for (; s < s1; ++s) a[0] += p[(size_t)s * kBins];
        qsum[grp][lb] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    __syncthreads();
    if (grp == 0) {
        unsigned long long t = 0;
#pragma unroll
        for (uint32_t q = 0; q < kFinalizeSplit; ++q) t += qsum[q][lb];
        // carries of the packed counters (exact pass) may be negative; the total is not
        const long long c = spill[b] + (long long)t;
        spill[b] = 0;
        // device atomics: the accumulators may be shared by several shards, also by processes
        // on other GPUs through peer memory (prngd_ipc_open) -- the statistics reduction
        unsigned long long *h = reinterpret_cast<unsigned long long *>(d_hist);
        if (c) stat_add_u64<MC>(&h[b], (unsigned long long)c);
        local = c;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(~0u, local, o);
    if ((threadIdx.x & 31u) == 0) part[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
        stat_add_u64<MC>(reinterpret_cast<unsigned long long *>(d_count), (unsigned long long)t);
    }
    if (blockIdx.x == 0 && threadIdx.x < 4) {
        double acc = 0.0;
        for (int s = 0; s < n_slabs; ++s) acc = __dadd_rn(acc, pow_slab[s * 4 + threadIdx.x]);
        if (d_pow) stat_add_f64<MC>(&d_pow[threadIdx.x], acc);  // null: histogram-only call
    }
    if (arrive) {
        __threadfence_system();  // this thread's adds are performed before the block arrives
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(done, 1u) == gridDim.x - 1) {
            __threadfence_system();
            *done = 0u;  // stream-ordered: the next call's blocks start after this kernel
            red_release_sys_u64<MC>(arrive, 1ull);
        }
    }
}

static void finalize_launch(bool mc, cudaStream_t st, const uint32_t *slab, int n_slabs,
                            int64_t *spill, const double *pow_slab, int64_t *d_hist,
                            double *d_pow, int64_t *d_count, uint32_t *overflow, uint32_t *done,
                            unsigned long long *arrive) {
    constexpr unsigned kFinalizeBlocks = kBins / (256 / kFinalizeSplit);
    if (mc)
        finalize_kernel<true><<<kFinalizeBlocks, 256, 0, st>>>(slab, n_slabs, spill, pow_slab,
                                                               d_hist, d_pow, d_count, overflow,
                                                               done, arrive);
    else
        finalize_kernel<false><<<kFinalizeBlocks, 256, 0, st>>>(slab, n_slabs, spill, pow_slab,
                                                                d_hist, d_pow, d_count, overflow,
                                                                done, arrive);
}

// Device-side wait for the completion counter of prngd_generate_consume_ex (acquire, system
// scope).  Traps (a sticky launch error at the caller's next synchronisation) after timeout_ns.
__global__ void wait_arrivals_kernel(const unsigned long long *arrive, unsigned long long target,
                                     unsigned long long timeout_ns) {
    unsigned long long t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(arrive) : "memory");
        if (v >= target) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) __trap();
        __nanosleep(2000);
    }
}

cudaError_t launch_wait_arrivals(const unsigned long long *arrive, unsigned long long target,
                                 unsigned long long timeout_ns, cudaStream_t st) {
    wait_arrivals_kernel<<<1, 1, 0, st>>>(arrive, target, timeout_ns);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ NEXT-2 MRG32k3a
// Same ROW burst store, MRG32k3a base draws (ALU/latency-bound: ~2 x 25 integer ops per draw),
// so shorter bursts (smaller tiles) buy occupancy.
#ifndef PRNGD_MRG_RC
#define PRNGD_MRG_RC 16  // A/B on cfg3 shape (per-draw loops): 16 -> 136, 32 -> 129, 64 -> 119
#endif
constexpr int kMrgCols = PRNGD_MRG_RC;
constexpr size_t kMrgTileBytes = (size_t)32 * (kMrgCols * 8 + 16);
constexpr size_t kMrgStageBytes = PRNGD_MRG_STAGE == 0 ? kMrgTileBytes : 0;
template <bool EQ4, bool SAMEW, bool ALG1, bool SPECB = false>
__global__ void __launch_bounds__(32) gen_mrg_kernel(const __grid_constant__ GenArgs g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t row0 = (uint64_t)blockIdx.x * 32u;
    NoConsumer nc;
    // 256-byte alignment is all the rings need (no TMA here): a smaller footprint, more warps
    const uint32_t base = (smem_u32(smem_raw) + (kMrgRingBytes - 1)) & ~(kMrgRingBytes - 1);
    static_assert(kMrgTileBytes % kMrgRingBytes == 0, "rings must stay kMrgRingBytes aligned");
    MrgProducer2<EQ4, SAMEW, ALG1, SPECB, PRNGD_MRG_SWZ && PRNGD_MRG_STAGE != 2,
                 PRNGD_MRG_REGCONST != 0> prod(
        g, g.stream_begin + row0 + lane, base + (uint32_t)kMrgStageBytes + lane * kMrgRingBytes,
        lane);
    if constexpr (PRNGD_MRG_STAGE == 2) {
        // Every lane consumes exactly 128 bytes of its ring per batch, and its read counter
        // started at 16 * lane, so the bytes batch b consumed sit at (16 l + 128 b) mod 256 of
        // lane l's ring for every l: free until the next fill, they hold the lane's 16 outputs
        // while the warp writes the 32 x 128-byte tile row by row (16-byte chunks, 4 rows per
        // instruction).
        const uint32_t rings = base;
        const bool live = row0 + lane < g.n_streams;
        const bool full_rows = row0 + 32u <= g.n_streams;
        const bool vec = (g.nps % 2u) == 0u && (reinterpret_cast<uintptr_t>(g.out) & 15u) == 0u;
        const uint32_t c = lane & 7u, rsub = lane >> 3;
        double *dst = g.out + (row0 + lane) * g.nps;
        uint32_t boff = 0u;
#pragma unroll 1
        for (uint64_t col0 = 0; col0 < g.nps; col0 += kCols, boff ^= 128u) {
            double q[kCols];
            prod(q, g);
            if (vec && full_rows && col0 + kCols <= g.nps) {
                const uint32_t my = rings + lane * kMrgRingBytes, o0 = 16u * lane + boff;
#pragma unroll
                for (int k = 0; k < kCols / 2; ++k)
                    sts_v2(my | ((o0 + 16u * k) & 0xF0u), q[2 * k], q[2 * k + 1]);
                __syncwarp();
                double *d = g.out + (row0 + rsub) * g.nps + col0 + 2 * c;
#pragma unroll
                for (uint32_t r = rsub; r < 32u; r += 4u) {
                    double a, b;
                    lds_v2(rings + r * kMrgRingBytes + ((16u * r + boff + 16u * c) & 0xF0u), a, b);
                    stg_v2_cs(d, a, b);
                    d += 4u * g.nps;
                }
                __syncwarp();
            } else if (live) {
#pragma unroll
                for (int i = 0; i < kCols; ++i)
                    if (col0 + i < g.nps) dst[col0 + i] = q[i];
            }
        }
    } else if constexpr (PRNGD_MRG_STAGE == 1) {
        // each lane writes its own row straight from registers (16-byte stores); the L2 merges
        // the row's 128-byte lines before they reach HBM
        const bool live = row0 + lane < g.n_streams;
        double *dst = g.out + (row0 + lane) * g.nps;
        const bool vec = (g.nps % 2u) == 0u && (reinterpret_cast<uintptr_t>(g.out) & 15u) == 0u;
#pragma unroll 1
        for (uint64_t col0 = 0; col0 < g.nps; col0 += kCols) {
            double q[kCols];
            prod(q, g);
            if (!live) continue;
            if (vec && col0 + kCols <= g.nps) {
#pragma unroll
                for (int c = 0; c < kCols / 2; ++c) stg_v2_cs(dst + col0 + 2 * c, q[2 * c], q[2 * c + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < kCols; ++i)
                    if (col0 + i < g.nps) dst[col0 + i] = q[i];
            }
        }
    } else {
        run_rows_burst<false, kMrgCols>(g, base, lane, row0, prod, nc);
    }
}

// ------------------------------------------------------------------------------ NEXT-2 + S7 fused
// The fused consumer on the MRG32k3a base generator: persistent, one CTA per SM holding the
// 128 KiB packed histogram (the same optimistic adds, overflow check, exact pass and slabs as
// consume_kernel) and kMrgConsWarps warps, each with its lanes' 256-byte rings of valid draws.
// With outputs, a batch's 16 values are staged in the ring bytes the batch has just consumed
// (lane l consumed (16 l + 128 b) mod 256 of its ring, free until the next fill) and the warp
// writes the 32 x 128-byte tile row by row, so no separate tile is needed beside the histogram.
// Replaces "generate, then read the outputs back" (8 more bytes of HBM traffic per output and
// a second kernel) by ~11 instructions per output in the generator's epilogue.
#ifndef PRNGD_MRG_CONS_WARPS
#define PRNGD_MRG_CONS_WARPS 12
#endif
constexpr int kMrgConsWarps = PRNGD_MRG_CONS_WARPS;
constexpr size_t kMrgConsSmem = 1024 + (size_t)kHistWords * 4u + (size_t)kMrgConsWarps * 32u * kMrgRingBytes;
static_assert(kMrgRingBytes == 256u, "the in-ring staging assumes 256-byte rings");

template <bool EQ4, bool SAMEW, bool ALG1, bool SPECB, bool WRITE, bool RED, bool EXACT_GUARD>
__global__ void __launch_bounds__(kMrgConsWarps * 32, 1)
    consume_mrg_kernel(const __grid_constant__ GenArgs g) {
    if (EXACT_GUARD && *(volatile const uint32_t *)g.overflow == 0u) return;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = aligned_smem_base(smem_raw);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem_raw + (base - smem_u32(smem_raw)));
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t rings = base + kHistWords * 4u + warp * (32u * kMrgRingBytes);
    for (uint32_t i = threadIdx.x; i < kHistWords; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    ConsumerT<RED, false> cons;
    cons.init(hist, g.hist_spill, g.hist_only != 0u);
    const uint64_t n_tasks = (g.n_streams + 31u) / 32u;
    const bool vec = (g.nps % 2u) == 0u && (reinterpret_cast<uintptr_t>(g.out) & 15u) == 0u;
    const uint32_t c = lane & 7u, rsub = lane >> 3;
#pragma unroll 1
    for (uint64_t t = (uint64_t)blockIdx.x + (uint64_t)gridDim.x * warp; t < n_tasks;
         t += (uint64_t)gridDim.x * kMrgConsWarps) {
        const uint64_t row0 = t * 32u;
        MrgProducer2<EQ4, SAMEW, ALG1, SPECB, false, PRNGD_MRG_REGCONST_CONS != 0, kMrgStepCons> prod(g, g.stream_begin + row0 + lane,
                                                  rings + lane * kMrgRingBytes, lane, 16u);
        const bool live = row0 + lane < g.n_streams;
        const bool full_rows = row0 + 32u <= g.n_streams;
        double *dst = WRITE ? g.out + (row0 + lane) * g.nps : nullptr;
        uint32_t boff = 0u;
#pragma unroll 1
        for (uint64_t col0 = 0; col0 < g.nps; col0 += kCols, boff ^= 128u) {
            double q[kCols];
            prod(q, g);
            const bool full = col0 + kCols <= g.nps;
            if (live) {
                if (full) {
                    consume_batch(cons, q);
                } else {
#pragma unroll
                    for (int i = 0; i < kCols; ++i)
                        if (col0 + i < g.nps) cons.add(q[i], i);
                }
            }
            if constexpr (WRITE) {
                if (vec && full_rows && full) {
                    const uint32_t my = rings + lane * kMrgRingBytes, o0 = 16u * lane + boff;
#pragma unroll
                    for (int k = 0; k < kCols / 2; ++k)
                        sts_v2(my | ((o0 + 16u * k) & 0xF0u), q[2 * k], q[2 * k + 1]);
                    __syncwarp();
                    double *d = g.out + (row0 + rsub) * g.nps + col0 + 2 * c;
#pragma unroll
                    for (uint32_t r = rsub; r < 32u; r += 4u) {
                        double a, b;
                        lds_v2(rings + r * kMrgRingBytes + ((16u * r + boff + 16u * c) & 0xF0u), a, b);
                        stg_v2_cs(d, a, b);
                        d += 4u * g.nps;
                    }
                    __syncwarp();  // the staged bytes are read before the next fill reuses them
                } else if (live) {
#pragma unroll
                    for (int i = 0; i < kCols; ++i)
                        if (col0 + i < g.nps) dst[col0 + i] = q[i];
                }
            }
        }
    }
    unsigned long long expect = 0;
    if (RED && lane == 0)
        for (uint64_t t = (uint64_t)blockIdx.x + (uint64_t)gridDim.x * warp; t < n_tasks;
             t += (uint64_t)gridDim.x * kMrgConsWarps) {
            const uint64_t left = g.n_streams - t * 32u;
            expect += (left < 32u ? left : 32u) * g.nps;
        }
    consume_epilogue<RED, kMrgConsWarps>(cons, hist, g, expect);
}

// ------------------------------------------------------------------------------ NEXT-3 jump kernel
// One warp per stream, kJumpWarps streams per CTA.  Each round, lane l jumps the round-start
// state by l * 2P draws (J_l = T^(2P l), byte tables) and draws P consecutive pairs, keeping the
// outputs in registers; a warp scan of the per-lane accepted counts gives every accepted output
// its sequential position (pair-drop, R2), the lanes scatter them into a compact shared-memory
// run, and the warp writes the run with coalesced stores.  Lane 31's final state starts the next
// round; a short remainder is finished by one lane sequentially.  P = 17 (two rounds per
// 1024-output row, the short-row kernel) or P = kJumpPairsLong = 33 for rows of >= 1000 outputs:
// 1056 pairs cover a 1024-output row in ONE round unless more than 32 pairs are rejected (at
// w = 8, 8.3 expected), halving the jumps and scans per output; 128 registers, 4 CTAs per SM
// (cfg2, same box: 250.6 -> 273.4-273.6 Gd/s; 33 pairs unconstrained, 142 registers: 259;
// capped at 96 registers with spills: 251; 25 pairs: 223, `profiles/r02m_jump_pairs_ab.txt`).
constexpr int kJumpPairs = (int)(kJumpDraws / 2);
constexpr int kJumpPairsLong = 33;
#ifndef PRNGD_JUMP_LONG_MIN
#define PRNGD_JUMP_LONG_MIN 1000  // rows of at least this many outputs take the 33-pair rounds
#endif
#ifndef PRNGD_JUMP_TAIL
#define PRNGD_JUMP_TAIL 24
#endif
constexpr uint64_t kJumpTail = PRNGD_JUMP_TAIL;  // remainders up to this many finish on one lane
#ifndef PRNGD_JUMP_WARPS
#define PRNGD_JUMP_WARPS 4
#endif
constexpr int kJumpWarps = PRNGD_JUMP_WARPS;  // warps (streams) per CTA
// Compaction run of one round: output p at byte 8 (p + p / 16).  Lane l writes its i-th
// accepted output near p = 16 l + i, so without the pad every lane of a store hits the same
// bank (a 128-byte stride); with it they spread over the banks.  Reads of consecutive p stay
// contiguous within each run of 16.
// (An odd pair count spreads the lanes by itself: no pad.)
template <int P>
constexpr uint32_t jump_pad() { return (P % 2 == 0) ? 1u : 0u; }
template <int P>
constexpr uint32_t jump_comp_bytes() { return 32u * P * 8u + (32u * P / 16u + 2u) * 8u; }
template <int P>
__device__ __forceinline__ uint32_t jump_comp_off(uint32_t p) {
    return (p + jump_pad<P>() * (p >> 4)) << 3;
}

// Jump-kernel modes for Eq.(4) with w = 8 or 16 and both draws at full width (sh1 = sh2 =
// 32 - w, e.g. cfg2's top bytes): v = x1 2^w + x2 is the top w bits of d1 followed by the top w
// bits of d2, ONE byte permute (instead of two shifts, a wide multiply-add and a move), and
// converts exactly from 16 / 32 bits -- the same v, the same Eq.(4) operations, the same bits.
#ifndef PRNGD_JUMP_NARROW
#define PRNGD_JUMP_NARROW 1
#endif
constexpr int kJumpMode8 = 8, kJumpMode16 = 9;
template <bool W8>
__device__ __forceinline__ double eq4_narrow(uint32_t d1, uint32_t d2, const GenArgs &g) {
    double z;
    if (W8) {
        // bytes (d2.b3, d1.b3, d2.b0, d2.b0): the low 16 bits are v; convert them alone
        const uint32_t v = __byte_perm(d2, d1, 0x0073);
        asm("{\n\t.reg .u16 h;\n\tcvt.u16.u32 h, %1;\n\tcvt.rn.f64.u16 %0, h;\n\t}"
            : "=d"(z) : "r"(v));
    } else {
        z = __uint2double_rn(__byte_perm(d2, d1, 0x7632));  // (d1 >> 16) << 16 | d2 >> 16
    }
    const double n = __dsub_rn(z, g.Cs);
    const double q0 = __dmul_rn(n, g.y);  // Markstein, as eq4_scaled
    const double r = __fma_rn(-q0, g.Ds, n);
    return __fma_rn(r, g.y, q0);
}

__device__ __forceinline__ Xs128 jump_state(const uint4 *__restrict__ tab, const Xs128 &s) {
    const uint32_t words[4] = {s.x, s.y, s.z, s.w};
    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        const uint32_t v = (words[b >> 2] >> (8 * (b & 3))) & 0xFFu;
        const uint4 t = __ldg(&tab[b * 256 + v]);
        r0 ^= t.x;
        r1 ^= t.y;
        r2 ^= t.z;
        r3 ^= t.w;
    }
    return Xs128{r0, r1, r2, r3};
}

// The same jump through nibble tables: J * s = XOR over the 32 nibbles of s of tab[p][nibble].
__device__ __forceinline__ Xs128 jump_state_nib(const uint4 *__restrict__ tab, const Xs128 &s) {
    const uint32_t words[4] = {s.x, s.y, s.z, s.w};
    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        const uint32_t v = (words[p >> 3] >> (4 * (p & 7))) & 0xFu;
        const uint4 t = __ldg(&tab[p * 16 + v]);
        r0 ^= t.x;
        r1 ^= t.y;
        r2 ^= t.z;
        r3 ^= t.w;
    }
    return Xs128{r0, r1, r2, r3};
}

// J_l * s through the lane-interleaved byte tables ([b][v][lane], jump_tables_interleaved): the
// lanes that jump the same state s read one contiguous run per table row (16 x 16-byte loads).
__device__ __forceinline__ Xs128 jump_state_lane(const uint4 *__restrict__ tabs, const Xs128 &s,
                                                 uint32_t lane) {
    const uint32_t words[4] = {s.x, s.y, s.z, s.w};
    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t v = (words[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        const uint4 t = __ldg(&tabs[((uint32_t)k * 256u + v) * 32u + lane]);
        r0 ^= t.x;
        r1 ^= t.y;
        r2 ^= t.z;
        r3 ^= t.w;
    }
    return Xs128{r0, r1, r2, r3};
}

// Resident CTAs per SM the register budget must allow: 7 x 4 warps x 148 SMs = 4144 >= cfg2's
// 4096 streams, so cfg2 runs as ONE wave (74 registers gave 6 CTAs: 1.15 waves).
#ifndef PRNGD_JUMP_MINB
#define PRNGD_JUMP_MINB 1  // A/B cfg2: 7 (one wave, 72 regs + spills) 253 vs 1 (74 regs) 252 Gd/s
#endif
template <int MODE, int P>
__global__ void __launch_bounds__(kJumpWarps * 32, P > 32 ? 4 : PRNGD_JUMP_MINB)
    gen_jump_kernel(const GenArgs g, const uint4 *__restrict__ tabs) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t row = (uint64_t)blockIdx.x * kJumpWarps + warp;
    if (row >= g.n_streams) return;
    constexpr bool FULL32 = MODE == 2;
    constexpr bool EQ4 = MODE >= 1;
    constexpr bool NARROW = MODE == kJumpMode8 || MODE == kJumpMode16;
    const uint32_t sh1 = (MODE == 2 || MODE == 3) ? 0u : g.sh1, sh2 = FULL32 ? 0u : g.sh2;
    const uint32_t w = (MODE == 2 || MODE == 3) ? 32u : g.w;
    const uint32_t lo = FULL32 ? 1u : g.lo, span = FULL32 ? 0xFFFFFFFEu : g.span;
    // NARROW: the band test on the raw draw, x1 = d >> sh1 in [lo, lo + span) <=> d in
    // [lo 2^sh1, (lo + span) 2^sh1) (lo + span = a < 2^w, so no overflow)
    const uint32_t lo_s = NARROW ? lo << sh1 : 0u, span_s = NARROW ? span << sh1 : 0u;
    const uint32_t comp = aligned_smem_base(smem_raw) + warp * jump_comp_bytes<P>();

    double *row_out = g.out + row * g.nps;
    Xs128 S = stream_start(g.seed, g.stream_begin + row);
    uint64_t base = 0;
#pragma unroll 1
    while (base < g.nps) {
        // every lane jumps the same round-start state: with the lane index innermost in the
        // byte tables ([b][v][lane]) each of the 16 loads reads one contiguous 512-byte run
        Xs128 st = lane ? jump_state_lane(tabs, S, lane) : S;
        double q[P];
        using MaskT = typename std::conditional<(P > 32), uint64_t, uint32_t>::type;
        MaskT mask = 0;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if constexpr (NARROW) {
                const uint32_t d1 = draw(st);
                const uint32_t d2 = draw(st);
                mask |= (MaskT)(d1 - lo_s < span_s ? 1u : 0u) << i;
                q[i] = eq4_narrow<MODE == kJumpMode8>(d1, d2, g);
            } else {
                const uint32_t x1 = draw(st) >> sh1;
                const uint32_t x2 = draw(st) >> sh2;
                mask |= (MaskT)(accepted(x1, lo, span) ? 1u : 0u) << i;
                q[i] = EQ4 ? eq4_mode<MODE, false>(x1, x2, g)
                           : map_pair<false, true>(x1, x2, g.map);
            }
        }
        if (EQ4 && g.span != g.span_fast) {  // R11 clamp only where the host found it needed
#pragma unroll
            for (int i = 0; i < P; ++i) q[i] = fmin(q[i], kBelowOne);
        }
        const uint32_t cnt = P > 32 ? (uint32_t)__popcll(mask) : (uint32_t)__popc((uint32_t)mask);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        // compact: accepted output k of this lane at position incl - cnt + k of the round
        uint32_t pos = incl - cnt;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if ((mask >> i) & (MaskT)1) {
                sts_f64(comp + jump_comp_off<P>(pos), q[i]);
                ++pos;
            }
        }
        __syncwarp();
        // (16-byte copies of slot pairs, with the run shifted to the output's parity: more
        // registers, spills at P = 33, cfg2 255 vs 272 Gd/s -- not kept)
        const uint64_t n = (g.nps - base) < (uint64_t)total ? (g.nps - base) : (uint64_t)total;
        for (uint32_t j = lane; j < (uint32_t)n; j += 32u) {
            double v;
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(comp + jump_comp_off<P>(j)));
            row_out[base + j] = v;
        }
        __syncwarp();
        S.x = __shfl_sync(0xFFFFFFFFu, st.x, 31);
        S.y = __shfl_sync(0xFFFFFFFFu, st.y, 31);
        S.z = __shfl_sync(0xFFFFFFFFu, st.z, 31);
        S.w = __shfl_sync(0xFFFFFFFFu, st.w, 31);
        base += total;
        // A short remainder (rejections made the last round fall a few outputs short, e.g.
        // ~8 of 1024 at w = 8) is cheaper as a sequential tail on one lane than as a full round.
        const uint64_t rem = g.nps > base ? g.nps - base : 0;
        if (rem > 0 && rem <= kJumpTail) {
            if (lane == 0) {
                Xs128 t = S;
                for (uint64_t i = 0; i < rem; ++i)
                    row_out[base + i] = exact_output<EQ4, false, false>(t, sh1, sh2, w, lo, span, g);
            }
            break;
        }
    }
}

// NEXT-3 for the narrow modes (w = 8 / 16, both draws at full width: cfg2): the same rounds as
// gen_jump_kernel, but a lane keeps the 16 / 32-bit pair value v = x1 2^w + x2 of each draw
// pair instead of its double (P registers instead of 2P), the compaction run holds these u32
// values (4 B per output instead of 8), and Eq.(4) is evaluated in the copy-out, two outputs
// per lane and store.  That halves the registers and the shared memory per warp, so cfg2's 4096
// streams run as ONE wave (32 warps per SM) instead of 1.7 waves at 16 warps per SM.  Same
// pairs, same v, same operations: the same bits as gen_jump_kernel.
template <int P>
constexpr uint32_t jumpn_comp_bytes() { return (32u * P + 2u) * 4u; }
#ifndef PRNGD_JUMPN_MINB
#define PRNGD_JUMPN_MINB 8
#endif
template <bool W8>
__device__ __forceinline__ uint32_t narrow_v(uint32_t d1, uint32_t d2) {
    // W8: bytes (d2.b3, d1.b3) = v in the low 16 bits (the high half is not used); W16:
    // (d1 >> 16) << 16 | d2 >> 16
    return W8 ? __byte_perm(d2, d1, 0x0073) : __byte_perm(d2, d1, 0x7632);
}
template <bool W8, bool CLAMP>
__device__ __forceinline__ double eq4_narrow_v(uint32_t v, const GenArgs &g) {
    // exact conversion of v (W8: the low 16 bits of the word; its high half is not v), then
    // Eq.(4) as eq4_narrow
    double z;
    if (W8)
        asm("{\n\t.reg .u16 h;\n\tcvt.u16.u32 h, %1;\n\tcvt.rn.f64.u16 %0, h;\n\t}"
            : "=d"(z) : "r"(v));
    else
        z = __uint2double_rn(v);
    const double n = __dsub_rn(z, g.Cs);
    const double q0 = __dmul_rn(n, g.y);
    const double r = __fma_rn(-q0, g.Ds, n);
    const double q = __fma_rn(r, g.y, q0);
    return CLAMP ? fmin(q, kBelowOne) : q;  // R11 where the host found it needed
}
__device__ __forceinline__ void stg_v2(double *p, double a, double b) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

#ifndef PRNGD_JUMP_NARROW_V
#define PRNGD_JUMP_NARROW_V 1  // 0: the narrow modes run gen_jump_kernel<kJumpMode8/16> (A/B)
#endif
template <bool W8, bool CLAMP, int P>
__global__ void __launch_bounds__(kJumpWarps * 32, PRNGD_JUMPN_MINB)
    gen_jump_narrow_kernel(const GenArgs g, const uint4 *__restrict__ tabs) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t row = (uint64_t)blockIdx.x * kJumpWarps + warp;
    if (row >= g.n_streams) return;
    // band test on the raw draw: x1 = d >> sh1 in [lo, lo + span) <=> d in [lo 2^sh1,
    // (lo + span) 2^sh1)
    const uint32_t lo_s = g.lo << g.sh1, span_s = g.span << g.sh1;
    const uint32_t comp = ((smem_u32(smem_raw) + 15u) & ~15u) + warp * jumpn_comp_bytes<P>();

    double *row_out = g.out + row * g.nps;
    Xs128 S = stream_start(g.seed, g.stream_begin + row);
    uint64_t base = 0;
#pragma unroll 1
    while (base < g.nps) {
        // lane l starts at draw 2 P l of the round (lane-interleaved byte tables)
        Xs128 st = lane ? jump_state_lane(tabs, S, lane) : S;
        uint32_t v[P];
        using MaskT = typename std::conditional<(P > 32), uint64_t, uint32_t>::type;
        MaskT mask = 0;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const uint32_t d1 = draw(st);
            const uint32_t d2 = draw(st);
            mask |= (MaskT)(d1 - lo_s < span_s ? 1u : 0u) << i;
            v[i] = narrow_v<W8>(d1, d2);
        }
        const uint32_t cnt = P > 32 ? (uint32_t)__popcll(mask) : (uint32_t)__popc((uint32_t)mask);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        // output p of the round goes to global element row_out[base + p] and to slot p + j0 of
        // the run, j0 = 1 when that element is odd: output pairs (p, p + 1) with p = j0 (mod 2)
        // are then 8-byte aligned in the run and 16-byte aligned in the output
        const uint32_t j0 = (uint32_t)(((uintptr_t)(row_out + base) >> 3) & 1u);
        uint32_t slot = incl - cnt + j0;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const uint32_t bit = (uint32_t)(mask >> i) & 1u;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                         "@p st.shared.u32 [%0], %1;\n\t}" ::"r"(comp + 4u * slot), "r"(v[i]), "r"(bit)
                         : "memory");
            slot += bit;
        }
        __syncwarp();
        const uint32_t n = (g.nps - base) < (uint64_t)total ? (uint32_t)(g.nps - base) : total;
        double *out = row_out + base;
        if (n > 0) {
            const uint32_t npair = (n - j0) >> 1;  // full 16-byte pairs after the odd head
            double *dst = out + j0 + 2u * lane;
            uint32_t sa = comp + 8u * (lane + j0);
#pragma unroll 4
            for (uint32_t k = lane; k < npair; k += 32u, dst += 64, sa += 256u) {
                uint32_t a, b;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(sa) : "memory");
                stg_v2(dst, eq4_narrow_v<W8, CLAMP>(a, g), eq4_narrow_v<W8, CLAMP>(b, g));
            }
            if (lane == 0 && j0) {  // odd head (slot 1)
                uint32_t a;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a) : "r"(comp + 4u) : "memory");
                out[0] = eq4_narrow_v<W8, CLAMP>(a, g);
            }
            if (lane == 31 && ((n - j0) & 1u)) {  // odd tail: output n - 1, slot n - 1 + j0
                uint32_t a;
                asm volatile("ld.shared.u32 %0, [%1];"
                             : "=r"(a) : "r"(comp + 4u * (n - 1u + j0)) : "memory");
                out[n - 1u] = eq4_narrow_v<W8, CLAMP>(a, g);
            }
        }
        __syncwarp();
        S.x = __shfl_sync(0xFFFFFFFFu, st.x, 31);
        S.y = __shfl_sync(0xFFFFFFFFu, st.y, 31);
        S.z = __shfl_sync(0xFFFFFFFFu, st.z, 31);
        S.w = __shfl_sync(0xFFFFFFFFu, st.w, 31);
        base += total;
        const uint64_t rem = g.nps > base ? g.nps - base : 0;
        if (rem > 0 && rem <= kJumpTail) {  // short remainder: one lane, sequentially
            if (lane == 0) {
                Xs128 t = S;
                for (uint64_t i = 0; i < rem; ++i) {
                    uint32_t d1, d2;
                    do {
                        d1 = draw(t);
                        d2 = draw(t);
                    } while (!(d1 - lo_s < span_s));
                    row_out[base + i] = eq4_narrow_v<W8, CLAMP>(narrow_v<W8>(d1, d2), g);
                }
            }
            break;
        }
    }
}

// ------------------------------------------------------------------------------ SEG store path
// Row segments: a lane owns one 1 KiB segment (kSegOut = 128 outputs) of a row, so the S =
// nps / 128 lanes of a row write it side by side and each flush puts S 512-byte chunks, 1 KiB
// apart, into the same row (tools/segment_sweep.py: 7.09 vs 6.73 TB/s for cfg3's rows, 6.9 vs
// 6.2 TB/s for cfg4's).  Lane j of a row starts at pair j*128 = draw j*kSegDraws of its stream
// through the jump tables T^(256 l).  Under pair-drop that pair range is fixed whatever the
// earlier lanes reject, but the output positions are not: the fast path assumes no rejection
// (and no x1 = a - 1, the only row the R11 clamp can touch) and a warp vote at the end sends
// the whole warp to seg_exact(), which rewrites every output of its rows exactly.
#ifndef PRNGD_SEG_HALF
#define PRNGD_SEG_HALF 64
#endif
constexpr int kSegHalf = PRNGD_SEG_HALF;  // outputs per lane per flush (one 512-byte chunk)
constexpr uint32_t kSegRS = kSegHalf * 8u + 16u;  // padded tile row stride (bytes)

// How a lane reaches its segment start T^(256 j) s (A/B):
//   0 byte tables, direct J_j (16 loads), next task's loads prefetched across a batch
//   1 nibble tables, direct J_j (32 loads, 8 KiB per j)
//   2 nibble tables, J_j as the product of J_(2^k) over the set bits k of j (<= log2 S stages)
//   3 byte tables, direct J_j, no prefetch
//   4 byte tables with the lane index innermost ([b][v][l]): the S lanes of a row jump the same
//     state, so each load is one contiguous run per row; prefetched like 0
#ifndef PRNGD_SEG_JUMP
#define PRNGD_SEG_JUMP 4  // cfg3 A/B: 0 -> 577, 1 -> 544, 2 -> 645, 3 -> 575 Gd/s
#endif


template <int MODE, bool IEEE, int SO>
__device__ __forceinline__ void seg_exact(const GenArgs &g, Xs128 st, uint32_t j, uint32_t S,
                                          uint64_t row, bool live) {
    constexpr bool FULL32 = MODE == 2;
    constexpr bool EQ4 = MODE >= 1;
    const uint32_t sh1 = (MODE == 2 || MODE == 3) ? 0u : g.sh1, sh2 = FULL32 ? 0u : g.sh2;
    const uint32_t w = (MODE == 2 || MODE == 3) ? 32u : g.w;
    const uint32_t lo = FULL32 ? 1u : g.lo, span = FULL32 ? 0xFFFFFFFEu : g.span;
    const Xs128 seg0 = st;
    // pass 1: accepted pairs among this lane's kSegOut pairs
    uint32_t cnt = 0;
#pragma unroll 1
    for (uint32_t i = 0; i < (uint32_t)SO; ++i) {
        const uint32_t x1 = draw(st) >> sh1;
        draw(st);
        cnt += accepted(x1, lo, span) ? 1u : 0u;
    }
    // exclusive scan over the S lanes of the row: first output position of this segment
    uint32_t incl = cnt;
    for (uint32_t o = 1; o < S; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o, S);
        if (j >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, S - 1, S);
    // pass 2: each accepted pair at its sequential position (the R11 clamp included)
    st = seg0;
    uint32_t pos = incl - cnt;
    double *row_out = g.out + row * g.nps;
#pragma unroll 1
    for (uint32_t i = 0; i < (uint32_t)SO; ++i) {
        const uint32_t x1 = draw(st) >> sh1;
        const uint32_t x2 = draw(st) >> sh2;
        if (accepted(x1, lo, span)) {
            const double q = EQ4 ? eq4_pair<IEEE, true>(x1, x2, w, g.Cs, g.Ds, g.y)
                                 : map_pair<IEEE, true>(x1, x2, g.map);
            if (live) row_out[pos] = q;
            ++pos;
        }
    }
    // the row's last lane continues the sequence past pair nps for the outputs still missing
    if (j == S - 1) {
#pragma unroll 1
        for (uint64_t p = total; p < g.nps; ++p) {
            const double q = exact_output<EQ4, IEEE, false>(st, sh1, sh2, w, lo, span, g);
            if (live) row_out[p] = q;
        }
    }
}

// Lane j's segment start T^(256 j) s from its stream start s (PRNGD_SEG_JUMP selects how).
__device__ __forceinline__ Xs128 seg_jump(const uint4 *__restrict__ tabs,
                                          const uint4 *__restrict__ my_tab, uint32_t j,
                                          uint32_t log2S, Xs128 s) {
#if PRNGD_SEG_JUMP == 0 || PRNGD_SEG_JUMP == 3
    (void)tabs, (void)log2S;
    return j ? jump_state(my_tab, s) : s;
#elif PRNGD_SEG_JUMP == 4
    (void)my_tab, (void)log2S;
    return j ? jump_state_lane(tabs, s, j) : s;
#elif PRNGD_SEG_JUMP == 1
    (void)tabs, (void)log2S;
    return j ? jump_state_nib(my_tab, s) : s;
#else
    (void)my_tab;
    for (uint32_t k = 0; k < log2S; ++k)
        if ((j >> k) & 1u) s = jump_state_nib(tabs + (size_t)(1u << k) * 32 * 16, s);
    return s;
#endif
}

// One batch of kCols outputs of the fast path into tile row `my` (row stride kSegRS: padded by
// 16 bytes, so lane writes and per-row flush reads are conflict-free).
template <int MODE, bool IEEE>
__device__ __forceinline__ void seg_batch(Xs128 &st, bool &rej, uint32_t my, uint32_t b,
                                          uint32_t lane, const GenArgs &g) {
    constexpr bool FULL32 = MODE == 2;
    constexpr bool EQ4 = MODE >= 1;
    const uint32_t sh1 = (MODE == 2 || MODE == 3) ? 0u : g.sh1, sh2 = FULL32 ? 0u : g.sh2;
    const uint32_t lo = FULL32 ? 1u : g.lo;
    const uint32_t span_fast = FULL32 ? 0xFFFFFFFDu : g.span_fast;
    double q[kCols];
#pragma unroll
    for (int i = 0; i < kCols; ++i) {
        const uint32_t x1 = draw(st) >> sh1;
        const uint32_t x2 = draw(st) >> sh2;
        rej |= !accepted(x1, lo, span_fast);
        q[i] = EQ4 ? eq4_mode<MODE, IEEE>(x1, x2, g) : map_pair<IEEE, false>(x1, x2, g.map);
    }
#pragma unroll
    for (int c = 0; c < kCols / 2; ++c)
        sts_v2(my + ((b * (kCols / 2) + c) << 4), q[2 * c], q[2 * c + 1]);
}

// Row-segment layout of the fused consumer (Store::SEG with S7): a warp-task is 32 / S rows of
// nps = 128 S outputs, lane j of a row owns its pairs [128 j, 128 j + 128) and starts there by
// jump-ahead, so each 16-output batch flush writes 32 chunks of 128 bytes 1 KiB apart inside one
// contiguous 32 KiB block (pure-store ceiling 6.12 vs 5.31 TB/s for one lane per row,
// profiles/r02f_consumer_store_patterns.json), from the same 4.6 KiB tile as the ROW layout.
// Speculation as in SEG: a batch is computed assuming every x1 is accepted and below a - 1; the
// warp vote comes BEFORE the batch is counted, so the statistics only ever see values of
// accepted pairs.  On an anomaly the warp finishes the task exactly: each lane counts its
// remaining pairs (statistics of the accepted ones, R11 clamp included), the row's last lane
// continues past pair nps for the outputs the rejections cost, and seg_exact rewrites the rows'
// outputs at their shifted positions.  The statistics are position-free, so nothing counted
// before the anomaly needs retracting.
template <int MODE, class Cons>
__device__ __forceinline__ void run_task_seg_consume(const GenArgs &g, uint32_t tile,
                                                     uint32_t lane, uint64_t t, Cons &cons) {
    constexpr bool FULL32 = MODE == 2;
    const uint32_t sh1 = (MODE == 2 || MODE == 3) ? 0u : g.sh1, sh2 = FULL32 ? 0u : g.sh2;
    const uint32_t w = (MODE == 2 || MODE == 3) ? 32u : g.w;
    const uint32_t lo = FULL32 ? 1u : g.lo, span = FULL32 ? 0xFFFFFFFEu : g.span;
    const uint32_t span_fast = FULL32 ? 0xFFFFFFFDu : g.span_fast;
    const uint32_t log2S = g.seg_log2, S = 1u << log2S, j = lane & (S - 1u);
    const uint32_t rpw = 32u >> log2S;
    const uint64_t row0 = t * rpw, row = row0 + (lane >> log2S);
    const bool live = row < g.n_streams;
    const uint64_t rows_left = g.n_streams - row0;
    const uint32_t nchunks = rows_left >= rpw ? 32u : (uint32_t)rows_left << log2S;
    Xs128 st = stream_start(g.seed, g.stream_begin + row);
    if (j) st = jump_state_lane(g.jump_tab, st, j);  // T^(256 j) s (one run per row)
    const Xs128 seg0 = st;
    constexpr uint32_t RS = kCols * 8u + 16u;  // padded tile row (one batch per lane)
    const uint32_t my = tile + lane * RS;
    double *blk = g.out + row0 * g.nps;      // tile row r -> blk + 128 r + 16 b (nps = 128 S)
    constexpr uint32_t kB = (uint32_t)kSegOut / kCols;
    uint32_t b = 0;
#pragma unroll 1
    for (; b < kB; ++b) {
        const Xs128 save = st;
        double q[kCols];
        bool rej = false;
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
            const uint32_t x1 = draw(st) >> sh1;
            const uint32_t x2 = draw(st) >> sh2;
            rej |= !accepted(x1, lo, span_fast);
            q[i] = eq4_mode<MODE, false>(x1, x2, g);
        }
        if (__builtin_expect(__any_sync(0xFFFFFFFFu, rej), 0)) {
            st = save;
            break;
        }
        if (live) consume_batch(cons, q);
#pragma unroll
        for (int c = 0; c < kCols / 2; ++c) sts_v2(my + (c << 4), q[2 * c], q[2 * c + 1]);
        __syncwarp();
        const uint32_t c = lane & 7u, rsub = lane >> 3;
        double *dst = blk + (uint64_t)rsub * kSegOut + b * kCols + 2 * c;
        if (nchunks == 32u) {
#pragma unroll
            for (uint32_t r = rsub; r < 32u; r += 4u) {
                double a0, a1;
                lds_v2(tile + r * RS + (c << 4), a0, a1);
                stg_v2_cs(dst, a0, a1);
                dst += 4u * kSegOut;
            }
        } else {
#pragma unroll 1
            for (uint32_t r = rsub; r < nchunks; r += 4u) {
                double a0, a1;
                lds_v2(tile + r * RS + (c << 4), a0, a1);
                stg_v2_cs(dst, a0, a1);
                dst += 4u * kSegOut;
            }
        }
        __syncwarp();
    }
    if (__builtin_expect(b < kB, 0)) {  // warp-uniform: the vote above
        // statistics of this lane's remaining pairs, exactly (R11 clamp included)
        uint32_t cnt = b * (uint32_t)kCols;  // every earlier pair was accepted
#pragma unroll 1
        for (uint32_t i = b * (uint32_t)kCols; i < (uint32_t)kSegOut; ++i) {
            const uint32_t x1 = draw(st) >> sh1;
            const uint32_t x2 = draw(st) >> sh2;
            if (accepted(x1, lo, span)) {
                if (live) cons.add(eq4_pair<false, true>(x1, x2, w, g.Cs, g.Ds, g.y));
                ++cnt;
            }
        }
        uint32_t tot = cnt;  // the row's accepted pairs among its nps pairs
        for (uint32_t o = 1; o < S; o <<= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
        if (j == S - 1u) {   // the outputs the rejections cost, past pair nps
#pragma unroll 1
            for (uint64_t p = tot; p < g.nps; ++p) {
                const double q = exact_output<true, false, false>(st, sh1, sh2, w, lo, span, g);
                if (live) cons.add(q);
            }
        }
        __syncwarp();  // the speculative stores above come before the exact rewrite
        seg_exact<MODE, false, (int)kSegOut>(g, seg0, j, S, row, live);
    }
}

// One-warp CTAs (12 per SM, smem-bound), each running `tpc` consecutive warp tasks of 32
// lane segments (a task = 32 / S rows = one contiguous 32 KiB block of the output), so the
// hardware's in-order CTA dispatch keeps the blocks being written in one moving window (a
// persistent grid striding over tasks measured 752 vs 912 Gd/s on the same stores).  The jump
// of a lane's NEXT task is issued before the current task's first batch and folded in after
// it, so its 16 table loads (L2 latency) overlap generation; only the CTA's first jump is
// exposed.  The 64 registers the loads occupy are free at this occupancy.
// SO = outputs per lane segment (128 = 1 KiB; 64 / 32 for few-stream shapes, which gives more
// lanes per row and a shorter serial chain per lane).  F = outputs per flush.
template <int MODE, bool IEEE, int SO>
__global__ void __launch_bounds__(32, 12)
    gen_seg_kernel(const GenArgs g, const uint4 *__restrict__ tabs, uint32_t log2S,
                   uint64_t n_tasks, uint32_t tpc) {
    const uint64_t t_end0 = ((uint64_t)blockIdx.x + 1) * tpc;
    const uint64_t t_end = t_end0 < n_tasks ? t_end0 : n_tasks;
    extern __shared__ uint8_t smem_raw[];
    constexpr uint32_t F = SO < kSegHalf ? SO : kSegHalf;
    constexpr uint32_t RS = F * 8u + 16u;  // padded tile row stride
    constexpr uint32_t kBatchesPerFlush = F / kCols;
    constexpr uint32_t kBatches = SO / kCols;
    const uint32_t lane = threadIdx.x;
    const uint32_t S = 1u << log2S;            // lanes (segments) per row
    const uint32_t j = lane & (S - 1u);        // this lane's segment
    const uint32_t rloc = lane >> log2S;       // this lane's row within the task
    const uint32_t rows_per_warp = 32u >> log2S;
#if PRNGD_SEG_JUMP == 1 || PRNGD_SEG_JUMP == 2
    const uint4 *my_tab = tabs + (size_t)j * 32 * 16;   // nibble tables, 8 KiB per lane matrix
#else
    const uint4 *my_tab = tabs + (size_t)j * 16 * 256;  // byte tables, 64 KiB per lane matrix
#endif
    const uint32_t tile = aligned_smem_base(smem_raw);
    const uint32_t my = tile + lane * RS;  // this lane's tile row
    uint64_t t = (uint64_t)blockIdx.x * tpc;
    Xs128 st = stream_start(g.seed, g.stream_begin + t * rows_per_warp + rloc);
    st = seg_jump(tabs, my_tab, j, log2S, st);
#pragma unroll 1
    for (; t < t_end; ++t) {
        const uint64_t row0 = t * rows_per_warp;
        const uint64_t row = row0 + rloc;
        const bool live = row < g.n_streams;
        // tile rows that belong to existing rows: all 32 except in a ragged last task
        const uint64_t rows_left = g.n_streams - row0;
        const uint32_t nchunks = rows_left >= rows_per_warp ? 32u : (uint32_t)rows_left << log2S;
        const Xs128 seg0 = st;
        // next task's start state: S1 now, its jump loads in flight during the first batch
        const uint64_t tn = t + 1;
        Xs128 nxt = stream_start(g.seed, g.stream_begin + tn * rows_per_warp + rloc);
        const bool jump_next = j != 0 && tn < t_end;
        uint4 pf[16];
#if PRNGD_SEG_JUMP == 0 || PRNGD_SEG_JUMP == 4
        if (jump_next) {
            const uint32_t words[4] = {nxt.x, nxt.y, nxt.z, nxt.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint32_t v = (words[k >> 2] >> (8 * (k & 3))) & 0xFFu;
                pf[k] = PRNGD_SEG_JUMP == 4 ? __ldg(&tabs[((uint32_t)k * 256u + v) * 32u + j])
                                            : __ldg(&my_tab[k * 256 + v]);
            }
        }
#endif
        bool rej = false;
        seg_batch<MODE, IEEE>(st, rej, my, 0, lane, g);
#if PRNGD_SEG_JUMP == 0 || PRNGD_SEG_JUMP == 4
        if (jump_next) {
            uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                r0 ^= pf[k].x;
                r1 ^= pf[k].y;
                r2 ^= pf[k].z;
                r3 ^= pf[k].w;
            }
            nxt = Xs128{r0, r1, r2, r3};
        }
#else
        if (tn < t_end) nxt = seg_jump(tabs, my_tab, j, log2S, nxt);
#endif
#pragma unroll 1
        for (uint32_t k = 1; k <= kBatches; ++k) {
            if (k % kBatchesPerFlush == 0) {
                // flush: tile row r (segment r of the task) -> F outputs at (row0 + r / S) * nps
                // + (r % S) * SO + h * F = row0 * nps + r * SO + h * F (nps = SO * S): the task
                // is one contiguous block, lane segments SO outputs apart.  One instruction
                // writes 64 outputs (512 B): 64 / F tile rows, lane l at element 2 l of them.
                const uint32_t h = k / kBatchesPerFlush - 1;
                __syncwarp();
                double *base = g.out + row0 * g.nps + h * F;
                const uint32_t ninstr = nchunks * F / 64u;
#pragma unroll 4
                for (uint32_t i = 0; i < ninstr; ++i) {
                    const uint32_t e = i * 64u + 2u * lane;  // element of the flushed block
                    const uint32_t r = e / F, c = (e % F) / 2u;
                    double a, b2;
                    lds_v2(tile + r * RS + (c << 4), a, b2);
                    stg_v2_cs(base + (uint64_t)r * SO + (e % F), a, b2);
                }
                __syncwarp();
            }
            if (k < kBatches) seg_batch<MODE, IEEE>(st, rej, my, k % kBatchesPerFlush, lane, g);
        }
        if (__builtin_expect(__any_sync(0xFFFFFFFFu, rej), 0)) {
            __syncwarp();  // the speculative stores above are ordered before the exact rewrite
            seg_exact<MODE, IEEE, SO>(g, seg0, j, S, row, live);
        }
        st = nxt;
    }
}

// ------------------------------------------------------------------------------ SEGC store path
// Column blocks: a CTA of kSegcWarps = 8 warps owns a task of 32 consecutive rows (one 256 KiB
// block of the output for cfg3); lane r of every warp generates row row0 + r, and warp j owns
// column block j (L = nps / 8 outputs) of all 32 rows.  Lane (j, r) starts at pair j * L of its
// stream through J_j = T^(2 L j), applied with nibble tables held in shared memory (56 KiB,
// loaded once per persistent CTA); because j is warp-uniform every lane of a warp reads the same
// table.  Each warp flushes 512-byte row chunks exactly like the ROW kernel, but the CTA
// completes its 32-row block in L / 64 flushes instead of nps / 64 (tools/rot_sweep.py
// blockcol: 7.1 vs 6.7 TB/s for cfg3's rows, 6.6 vs 6.0 TB/s for cfg4's).
// Rejection (and x1 = a - 1, the R11 clamp row) is speculated away; the warps flag their rows
// in a per-task mask and, after the task's barrier, flagged rows are rewritten exactly: every
// warp recounts its block's accepted pairs, a prefix over the 8 blocks (shared memory) places
// each accepted output, and warp 7 continues the stream past pair nps for the missing tail.
constexpr int kSegcWarps = 8;
constexpr int kSegcTabBytes = (kSegcWarps - 1) * 32 * 16 * 16;  // J_1..J_7 nibble tables, 56 KiB

__device__ __forceinline__ Xs128 jump_state_nib_smem(uint32_t tab, const Xs128 &s) {
    const uint32_t words[4] = {s.x, s.y, s.z, s.w};
    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        const uint32_t v = (words[p >> 3] >> (4 * (p & 7))) & 0xFu;
        uint32_t a, b, c, d;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                     : "r"(tab + (uint32_t)(p * 16 + v) * 16u));
        r0 ^= a;
        r1 ^= b;
        r2 ^= c;
        r3 ^= d;
    }
    return Xs128{r0, r1, r2, r3};
}

template <int MODE, bool IEEE>
__device__ __noinline__ void segc_exact(const GenArgs &g, Xs128 st, uint32_t j, uint32_t lane,
                                        uint64_t row, bool fix, uint32_t L, uint32_t *cnt) {
    constexpr bool FULL32 = MODE == 2;
    constexpr bool EQ4 = MODE >= 1;
    const uint32_t sh1 = (MODE == 2 || MODE == 3) ? 0u : g.sh1, sh2 = FULL32 ? 0u : g.sh2;
    const uint32_t w = (MODE == 2 || MODE == 3) ? 32u : g.w;
    const uint32_t lo = FULL32 ? 1u : g.lo, span = FULL32 ? 0xFFFFFFFEu : g.span;
    const Xs128 seg0 = st;
    if (fix) {  // pass 1: accepted pairs among this block's L pairs
        uint32_t c = 0;
        for (uint32_t i = 0; i < L; ++i) {
            const uint32_t x1 = draw(st) >> sh1;
            draw(st);
            c += accepted(x1, lo, span) ? 1u : 0u;
        }
        cnt[j * 32 + lane] = c;
    }
    __syncthreads();
    if (fix) {
        uint32_t pos = 0, total = 0;
        for (uint32_t i = 0; i < (uint32_t)kSegcWarps; ++i) {
            const uint32_t c = cnt[i * 32 + lane];
            pos += i < j ? c : 0u;
            total += c;
        }
        // pass 2: every accepted pair at its sequential position (R11 clamp included)
        st = seg0;
        double *row_out = g.out + row * g.nps;
        for (uint32_t i = 0; i < L; ++i) {
            const uint32_t x1 = draw(st) >> sh1;
            const uint32_t x2 = draw(st) >> sh2;
            if (accepted(x1, lo, span)) {
                row_out[pos++] = EQ4 ? eq4_pair<IEEE, true>(x1, x2, w, g.Cs, g.Ds, g.y)
                                     : map_pair<IEEE, true>(x1, x2, g.map);
            }
        }
        if (j == kSegcWarps - 1)  // the row's last block continues past pair nps
            for (uint64_t p = total; p < g.nps; ++p)
                row_out[p] = exact_output<EQ4, IEEE, false>(st, sh1, sh2, w, lo, span, g);
    }
    __syncthreads();  // cnt is reused by the next rewrite
}

template <int MODE, bool IEEE>
__global__ void __launch_bounds__(kSegcWarps * 32, 1)
    gen_segc_kernel(const GenArgs g, const uint4 *__restrict__ tabs, uint64_t n_tasks) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint32_t cnt[kSegcWarps * 32];
    __shared__ uint32_t mask[3];
    const uint32_t lane = threadIdx.x & 31u, j = threadIdx.x >> 5;
    const uint32_t L = (uint32_t)(g.nps / kSegcWarps);  // outputs (pairs) per column block
    const uint32_t base = aligned_smem_base(smem_raw);
    const uint32_t tab_s = base;                                   // J_1..J_7, 8 KiB each
    const uint32_t tile = base + kSegcTabBytes + j * (32u * kSegRS);
    const uint32_t my = tile + lane * kSegRS;
    {   // nibble tables of J_1..J_7 (lane matrices 1..7 of the global table) into smem
        const uint4 *src = tabs + 32 * 16;
        for (uint32_t i = threadIdx.x; i < (uint32_t)(kSegcTabBytes / 16); i += blockDim.x) {
            const uint4 v = src[i];
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(tab_s + i * 16u), "r"(v.x),
                         "r"(v.y), "r"(v.z), "r"(v.w)
                         : "memory");
        }
        if (threadIdx.x < 3) mask[threadIdx.x] = 0u;
    }
    __syncthreads();
    const uint32_t my_tab = tab_s + (j ? (j - 1u) : 0u) * (32u * 16u * 16u);
    uint32_t it = 0;
#pragma unroll 1
    for (uint64_t t = blockIdx.x; t < n_tasks; t += gridDim.x, ++it) {
        const uint64_t row0 = t * 32u;
        const uint64_t row = row0 + lane;
        const bool live = row < g.n_streams;
        const uint64_t rows_left = g.n_streams - row0;
        const uint32_t nrows = rows_left < 32u ? (uint32_t)rows_left : 32u;
        Xs128 st = stream_start(g.seed, g.stream_begin + row);
        if (j) st = jump_state_nib_smem(my_tab, st);
        const Xs128 seg0 = st;
        bool rej = false;
        double *blk = g.out + row0 * g.nps + (uint64_t)j * L + 2 * lane;
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < L; c0 += kSegHalf) {
#pragma unroll 1
            for (uint32_t b = 0; b < (uint32_t)(kSegHalf / kCols); ++b)
                seg_batch<MODE, IEEE>(st, rej, my, b, lane, g);
            __syncwarp();
            // one 512-byte chunk of row r per instruction (32 lanes x 16 B)
            double *dst = blk + c0;
#pragma unroll 4
            for (uint32_t r = 0; r < nrows; ++r) {
                double a, b2;
                lds_v2(tile + r * kSegRS + (lane << 4), a, b2);
                stg_v2_cs(dst + (uint64_t)r * g.nps, a, b2);
            }
            __syncwarp();
        }
        const uint32_t flagged = __ballot_sync(0xFFFFFFFFu, rej && live);
        if (lane == 0 && flagged) atomicOr(&mask[it % 3], flagged);
        __syncthreads();  // also orders the speculative stores before any rewrite
        const uint32_t m = mask[it % 3];
        if (threadIdx.x == 0) mask[(it + 2) % 3] = 0u;  // read by everyone before barrier it
        if (__builtin_expect(m != 0u, 0))
            segc_exact<MODE, IEEE>(g, seg0, j, lane, row, live && ((m >> lane) & 1u), L, cnt);
    }
}

// ------------------------------------------------------------------------------ debug kernels
__global__ void debug_raw_kernel(const GenArgs g, uint32_t *raw, uint64_t draws) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n_streams) return;
    Xs128 st = stream_start(g.seed, g.stream_begin + i);
    for (uint64_t d = 0; d < draws; ++d) raw[i * draws + d] = draw(st);
}

template <bool ALG1>
__global__ void debug_pairs_kernel(const GenArgs g, uint32_t *pidx, uint64_t *consumed) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n_streams) return;
    Xs128 st = stream_start(g.seed, g.stream_begin + i);
    uint64_t p = 0;  // draws (ALG1) or pairs (R2) consumed
    for (uint64_t j = 0; j < g.nps; ++j) {
        uint32_t x1;
        if (ALG1) {
            do {
                x1 = draw(st) >> g.sh1;
                ++p;
            } while (!accepted(x1, g.lo, g.span));
            draw(st);
            ++p;
            if (pidx) pidx[i * g.nps + j] = (uint32_t)(p - 2);  // index of the accepted x1 draw
        } else {
            do {
                x1 = draw(st) >> g.sh1;
                draw(st);
                ++p;
            } while (!accepted(x1, g.lo, g.span));
            if (pidx) pidx[i * g.nps + j] = (uint32_t)(p - 1);
        }
    }
    if (consumed) consumed[i] = p;
}

template <bool IEEE>
__global__ void debug_map_kernel(const GenArgs g, const uint32_t *x1, const uint32_t *x2,
                                 double *z, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        z[i] = map_pair<IEEE, true>(x1[i], x2[i], g.map);
}

__global__ void debug_div_check_kernel(const GenArgs g, uint64_t n, uint64_t seed,
                                       unsigned long long *mismatch) {
    unsigned long long bad = 0;
    const uint32_t m1 = g.sh1 >= 32 ? 0u : (0xFFFFFFFFu >> g.sh1);
    const uint32_t m2 = g.sh2 >= 32 ? 0u : (0xFFFFFFFFu >> g.sh2);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = splitmix_finalize(seed + (i + 1) * kGamma);
        uint32_t x1 = (uint32_t)h & m1, x2 = (uint32_t)(h >> 32) & m2;
        // a quarter of the samples hug the top and bottom of x1 (where R11 and tiny q live)
        if ((i & 3u) == 1u) x1 = m1 - (x1 & 7u);
        if ((i & 3u) == 2u) x1 = x1 & 7u;
        const uint64_t v = ((uint64_t)x1 << g.w) | (uint64_t)x2;
        const double fast = eq4_scaled<false, false>(v, g.Cs, g.Ds, g.y);
        const double ieee = eq4_scaled<true, false>(v, g.Cs, g.Ds, g.y);
        bad += (__double_as_longlong(fast) != __double_as_longlong(ieee)) ? 1ull : 0ull;
    }
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(~0u, bad, o);
    if ((threadIdx.x & 31u) == 0 && bad) atomicAdd(mismatch, bad);
}

// ------------------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static std::once_flag once;
    static EncodeTiledFn fn = nullptr;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// Tensor map over out[n_streams][nps] (doubles), box 16 columns x box_rows rows, 128B swizzle.
static cudaError_t make_tmap(CUtensorMap *m, double *out, uint64_t n_streams, uint64_t nps,
                             uint32_t box_rows) {
    std::memset(m, 0, sizeof(*m));
    EncodeTiledFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {nps, n_streams};
    const cuuint64_t strides[1] = {nps * 8u};
    const cuuint32_t box[2] = {(cuuint32_t)kCols, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// The dynamic shared-memory opt-in of a kernel, set once per (kernel, device): every kernel
// instantiation always launches with the same size, and the attribute call costs host time on
// the launch path of the small configurations.
template <class K>
static cudaError_t set_smem(K kernel, size_t bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const std::pair<const void *, int> key{reinterpret_cast<const void *>(kernel), dev};
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

template <int MODE, bool SPEC, bool IEEE, bool ALG1, Store ST>
static cudaError_t gen_launch(const CUtensorMap &m, const GenArgs &g, cudaStream_t st) {
    auto k = gen_kernel<MODE, SPEC, IEEE, ALG1, ST>;
    const size_t smem = gen_smem<ST>();
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    const uint64_t tasks = (g.n_streams + 31u) / 32u;
    const uint64_t grid = (tasks + gen_warps<ST>() - 1) / gen_warps<ST>();
    if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    k<<<(unsigned)grid, gen_warps<ST>() * 32, smem, st>>>(m, g);
    return cudaGetLastError();
}

template <Store ST>
static cudaError_t gen_dispatch_static(const CUtensorMap &m, const GenArgs &g, int mode,
                                       cudaStream_t st) {
    switch (mode - kModeStatic) {
#define PRNGD_STATIC(C) case C: return gen_launch<kModeStatic + C, true, false, false, ST>(m, g, st);
        PRNGD_STATIC(2) PRNGD_STATIC(3) PRNGD_STATIC(4) PRNGD_STATIC(5) PRNGD_STATIC(6)
        PRNGD_STATIC(7) PRNGD_STATIC(8) PRNGD_STATIC(9) PRNGD_STATIC(10) PRNGD_STATIC(11)
#undef PRNGD_STATIC
        default: return gen_launch<0, true, false, false, ST>(m, g, st);
    }
}

template <Store ST>
static cudaError_t gen_dispatch_store(const CUtensorMap &m, const GenArgs &g, const Plan &pl,
                                      int mode, cudaStream_t st) {
    if constexpr (ST == Store::ROW) {
        if (mode >= kModeStatic && pl.spec && !pl.ieee_div && !pl.alg1)
            return gen_dispatch_static<ST>(m, g, mode, st);
    }
    if (pl.spec && !pl.ieee_div && !pl.alg1) {
        if (mode == 2) return gen_launch<2, true, false, false, ST>(m, g, st);
        if (mode == 3) return gen_launch<3, true, false, false, ST>(m, g, st);
        if (mode == 1) return gen_launch<1, true, false, false, ST>(m, g, st);
    }
    if (pl.alg1)
        return pl.ieee_div ? gen_launch<0, false, true, true, ST>(m, g, st)
                           : gen_launch<0, false, false, true, ST>(m, g, st);
    if (pl.spec)
        return pl.ieee_div ? gen_launch<0, true, true, false, ST>(m, g, st)
                           : gen_launch<0, true, false, false, ST>(m, g, st);
    return pl.ieee_div ? gen_launch<0, false, true, false, ST>(m, g, st)
                       : gen_launch<0, false, false, false, ST>(m, g, st);
}

// Kernel specialisation: 2 = w = 32 full range Eq.(4) closed, 1 = Eq.(4) closed, 0 = generic.
static int kernel_mode(const GenArgs &g) {
    const bool eq4 = g.map.kind == 4 && g.map.open == 0;
    const bool full32 = eq4 && g.w == 32 && g.sh1 == 0 && g.sh2 == 0 && g.lo == 1u &&
                        g.span == 0xFFFFFFFEu && g.span_fast == 0xFFFFFFFDu;
    const bool w32 = eq4 && g.w == 32 && g.sh1 == 0;
    // MODE 1 composes v with one wide multiply-add and needs w <= 31; w = 32 with a narrower
    // x1 (rare) takes the generic kernel
    if (full32) return 2;
    if (w32) return 3;
    if (eq4) return g.w <= 31 ? 1 : 0;
    // the other mappings: compile-time mapping on the bulk ROW path (w = 32 needs sh1 = 0 for
    // the register-pair composition of x1 - sub)
    const int k = g.map.kind == 5 ? 1 : (g.map.kind == 6 ? 2 : 0);
    if (g.w == 32 && g.sh1 != 0) return 0;
    return kModeStatic + 4 * k + 2 * (g.map.open ? 1 : 0) + (g.w == 32 ? 1 : 0);
}

cudaError_t launch_generate(const GenArgs &g, const Plan &pl, cudaStream_t st, int) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    Store s = pl.store;
    const int f32 = kernel_mode(g);
#if PRNGD_AB_STORES
    if (s == Store::TMA && make_tmap(&m, g.out, g.n_streams, g.nps, 32u * kGenWarps) != cudaSuccess)
        s = Store::STG16;  // descriptor refused: fall back to coalesced st.global (same bits)
    switch (s) {
        case Store::ROW1K: return gen_dispatch_store<Store::ROW1K>(m, g, pl, f32, st);
        case Store::DIRECT: return gen_dispatch_store<Store::DIRECT>(m, g, pl, f32, st);
        case Store::TMA: return gen_dispatch_store<Store::TMA>(m, g, pl, f32, st);
        case Store::STG16: return gen_dispatch_store<Store::STG16>(m, g, pl, f32, st);
        default: break;
    }
#endif
    // product paths: 512-byte row bursts, or 8-byte stores for an unaligned output / odd nps
    return s == Store::ROW ? gen_dispatch_store<Store::ROW>(m, g, pl, f32, st)
                           : gen_dispatch_store<Store::STG8>(m, g, pl, f32, st);
}

// slabs (one u32 per bin per CTA), carry array, per-CTA power sums, then 16 bytes: the overflow
// flag and the finalize kernel's block-arrival counter (both zero between calls)
size_t consume_scratch_bytes(int num_sms) {
    return (size_t)num_sms * kBins * 4u + 65536u * 8u + (size_t)num_sms * 4u * 8u + 16u;
}
static void scratch_layout(GenArgs &g, void *scratch, int num_sms) {
    uint8_t *sp = static_cast<uint8_t *>(scratch);
    const size_t slabs = (size_t)num_sms * kBins * 4u;
    g.hist_slab = reinterpret_cast<uint32_t *>(sp);
    g.hist_spill = reinterpret_cast<int64_t *>(sp + slabs);
    g.pow_slab = reinterpret_cast<double *>(sp + slabs + 65536u * 8u);
    g.overflow = reinterpret_cast<uint32_t *>(sp + slabs + 65536u * 8u + (size_t)num_sms * 4u * 8u);
}

template <int MODE, bool SPEC, bool IEEE, bool ALG1, Store ST, bool WRITE, bool RED = false,
          bool EXACT_GUARD = false>
static cudaError_t cons_launch(const CUtensorMap &m, const GenArgs &g, int grid,
                               cudaStream_t st) {
    constexpr int kWarps = cons_warps<ST, WRITE>();
    auto k = consume_kernel<MODE, SPEC, IEEE, ALG1, ST, WRITE, RED, EXACT_GUARD>;
    const size_t smem = 1024 + (size_t)kHistWords * 4u +
                        (WRITE && (ST == Store::ROW || ST == Store::SEG)
                             ? (size_t)kWarps * 32 * (kConsRowCols * 8 + 16)
                             : (size_t)kWarps * ring<ST, WRITE>() * kTileBytes);
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kWarps * 32, smem, st>>>(m, g);
    return cudaGetLastError();
}

template <Store ST, bool WRITE, bool RED = false, bool EG = false>
static cudaError_t cons_dispatch(const CUtensorMap &m, const GenArgs &g, const Plan &pl,
                                 int mode, int grid, cudaStream_t st) {
    if (pl.spec && !pl.ieee_div && !pl.alg1) {
        if (mode == 2) return cons_launch<2, true, false, false, ST, WRITE, RED, EG>(m, g, grid, st);
        if (mode == 3) return cons_launch<3, true, false, false, ST, WRITE, RED, EG>(m, g, grid, st);
        if (mode == 1) return cons_launch<1, true, false, false, ST, WRITE, RED, EG>(m, g, grid, st);
    }
    if (pl.alg1)
        return pl.ieee_div ? cons_launch<0, false, true, true, ST, WRITE, RED, EG>(m, g, grid, st)
                           : cons_launch<0, false, false, true, ST, WRITE, RED, EG>(m, g, grid, st);
    if (pl.spec)
        return pl.ieee_div ? cons_launch<0, true, true, false, ST, WRITE, RED, EG>(m, g, grid, st)
                           : cons_launch<0, true, false, false, ST, WRITE, RED, EG>(m, g, grid, st);
    return pl.ieee_div ? cons_launch<0, false, true, false, ST, WRITE, RED, EG>(m, g, grid, st)
                       : cons_launch<0, false, false, false, ST, WRITE, RED, EG>(m, g, grid, st);
}

cudaError_t launch_generate_consume(const GenArgs &g0, const Plan &pl, double *d_out,
                                    int64_t *d_hist, double *d_pow, int64_t *d_count,
                                    unsigned long long *d_arrive, bool mc, void *scratch,
                                    size_t scratch_bytes, cudaStream_t st, int num_sms,
                                    int *launches) {
    *launches = 0;
    if (scratch_bytes < consume_scratch_bytes(num_sms)) return cudaErrorInvalidValue;
    GenArgs g = g0;
    g.hist_only = d_pow == nullptr ? 1u : 0u;
    g.out = d_out;
    scratch_layout(g, scratch, num_sms);
    const uint64_t tasks = (g.n_streams + 31u) / 32u;
    int grid = num_sms;  // persistent, one CTA per SM; every CTA gets a task when tasks >= grid
    if ((uint64_t)grid > tasks) grid = (int)tasks;
    if (grid < 1) grid = 1;
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const int f32 = kernel_mode(g);
    cudaError_t e;
    // Histogram adds are optimistic (RED, no carry tracking) unless the caller asked for the
    // exact carry path; an overflow found by the RED kernel triggers the exact pass (launched
    // always, returning at once when the flag is clear), which redoes every slab.
    const bool red = !pl.exact_hist;
    if (!d_out) {
        e = red ? cons_dispatch<Store::STG8, false, true>(m, g, pl, f32, grid, st)
                : cons_dispatch<Store::STG8, false>(m, g, pl, f32, grid, st);
    } else {
        Store s = pl.store;
        // row segments (SEG): the closed Eq.(4) kernels with speculation (rare rejection) only
        if (s == Store::SEG && !(pl.spec && !pl.ieee_div && !pl.alg1 && f32 >= 1 && f32 <= 3 &&
                                 g.nps % kSegOut == 0 && g.nps / kSegOut <= 32 &&
                                 ((g.nps / kSegOut) & (g.nps / kSegOut - 1)) == 0))
            s = Store::ROW;
        if (s == Store::SEG) {
            const void *tab = nullptr;
            if ((e = jump_tables_interleaved(kSegDraws, &tab)) != cudaSuccess) return e;
            g.jump_tab = static_cast<const uint4 *>(tab);
            g.seg_log2 = 0;
            while ((kSegOut << g.seg_log2) < g.nps) ++g.seg_log2;
            const uint64_t seg_tasks = (g.n_streams + (32u >> g.seg_log2) - 1) / (32u >> g.seg_log2);
            if ((uint64_t)grid > seg_tasks) grid = (int)seg_tasks;  // (>= the 32-row task count)
#define PRNGD_CONS_SEG(M)                                                                       \
    (red ? cons_launch<M, true, false, false, Store::SEG, true, true>(m, g, grid, st)            \
         : cons_launch<M, true, false, false, Store::SEG, true>(m, g, grid, st))
            e = f32 == 2 ? PRNGD_CONS_SEG(2) : f32 == 3 ? PRNGD_CONS_SEG(3) : PRNGD_CONS_SEG(1);
#undef PRNGD_CONS_SEG
        } else {
#define PRNGD_CONS_W(S)                                                                         \
    (red ? cons_dispatch<S, true, true>(m, g, pl, f32, grid, st)                                 \
         : cons_dispatch<S, true>(m, g, pl, f32, grid, st))
#if PRNGD_AB_STORES
        if (s == Store::TMA && make_tmap(&m, d_out, g.n_streams, g.nps, 32u) != cudaSuccess)
            s = Store::STG16;
        switch (s) {
            case Store::DIRECT: e = PRNGD_CONS_W(Store::DIRECT); break;
            case Store::TMA: e = PRNGD_CONS_W(Store::TMA); break;
            case Store::STG16: e = PRNGD_CONS_W(Store::STG16); break;
            default: e = (s == Store::ROW || s == Store::ROW1K) ? PRNGD_CONS_W(Store::ROW)
                                                                : PRNGD_CONS_W(Store::STG8);
        }
#else
        e = (s == Store::ROW || s == Store::ROW1K) ? PRNGD_CONS_W(Store::ROW)
                                                   : PRNGD_CONS_W(Store::STG8);
#endif
#undef PRNGD_CONS_W
        }
    }
    if (e != cudaSuccess) return e;
    *launches = 1;
    if (red) {  // exact fallback pass: consume-only (the outputs are already written)
        e = cons_dispatch<Store::STG8, false, false, true>(m, g, pl, f32, grid, st);
        if (e != cudaSuccess) return e;
        *launches = 2;
    }
    finalize_launch(mc, st, g.hist_slab, grid, g.hist_spill, g.pow_slab, d_hist,
                                         d_pow, d_count, g.overflow, g.overflow + 1, d_arrive);
    e = cudaGetLastError();
    if (e == cudaSuccess) *launches += 1;
    return e;
}

cudaError_t launch_consume_memory(const GenArgs &g0, const double *src, uint64_t n,
                                  int64_t *d_hist, double *d_pow, int64_t *d_count,
                                  unsigned long long *d_arrive, void *scratch,
                                  size_t scratch_bytes, cudaStream_t st, int num_sms,
                                  int *launches) {
    const bool mc = false;
    *launches = 0;
    if (scratch_bytes < consume_scratch_bytes(num_sms)) return cudaErrorInvalidValue;
    GenArgs g = g0;
    g.hist_only = d_pow == nullptr ? 1u : 0u;
    scratch_layout(g, scratch, num_sms);
    const int grid = num_sms;  // every CTA writes its slab (empty ones too): finalize reads all
    const size_t smem = 1024 + (size_t)kHistWords * 4u;
    cudaError_t e;
    if ((e = set_smem(hist_mem_kernel<true, false>, smem)) != cudaSuccess) return e;
    hist_mem_kernel<true, false><<<grid, kHistMemWarps * 32, smem, st>>>(src, n, g);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = set_smem(hist_mem_kernel<false, true>, smem)) != cudaSuccess) return e;
    hist_mem_kernel<false, true><<<grid, kHistMemWarps * 32, smem, st>>>(src, n, g);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    finalize_launch(mc, st, g.hist_slab, grid, g.hist_spill, g.pow_slab, d_hist,
                                         d_pow, d_count, g.overflow, g.overflow + 1, d_arrive);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches = 3;
    return cudaSuccess;
}

// The MRG32k3a kernel family of a parameter set (shared by the generator and the fused consumer)
struct MrgKind {
    bool eq4, samew, specb;
};
static MrgKind mrg_kind(const GenArgs &g, bool alg1) {
    MrgKind k;
    k.eq4 = g.map.kind == 4 && g.map.open == 0 && g.w <= 31;
    k.samew = g.mrg_t1 == g.mrg_t2 && g.mrg_mask1 == g.mrg_mask2;
    // band test per batch instead of per draw when fewer than 1 in 4096 x1 are out of band.
    // Alg. 1 drops a single draw, which shifts the x1/x2 roles of the later ones: only when
    // both have the same width (threshold and mask) is that harmless.
    const uint64_t range1 = (uint64_t)g.mrg_mask1 + 1u;
    k.specb = (range1 - g.span) * 4096u < range1 && (!alg1 || k.samew);
    return k;
}

// S1-S7 on MRG32k3a: fused pass (optimistic adds) + exact pass + finalize, as
// launch_generate_consume.
template <bool EQ4, bool SAMEW, bool ALG1, bool SPECB>
static cudaError_t cons_mrg_launch(const GenArgs &g, bool write, int grid, cudaStream_t st) {
    cudaError_t e;
#define PRNGD_CM(W, R, X)                                                                       \
    do {                                                                                        \
        auto k = consume_mrg_kernel<EQ4, SAMEW, ALG1, SPECB, W, R, X>;                          \
        if ((e = set_smem(k, kMrgConsSmem)) != cudaSuccess) return e;                          \
        k<<<grid, kMrgConsWarps * 32, kMrgConsSmem, st>>>(g);                                  \
        if ((e = cudaGetLastError()) != cudaSuccess) return e;                                  \
    } while (0)
    if (write)
        PRNGD_CM(true, true, false);
    else
        PRNGD_CM(false, true, false);
    PRNGD_CM(false, false, true);  // exact pass: returns at once unless a 16-bit field wrapped
#undef PRNGD_CM
    return cudaSuccess;
}

cudaError_t launch_generate_consume_mrg(const GenArgs &g0, bool alg1, double *d_out,
                                        int64_t *d_hist, double *d_pow, int64_t *d_count,
                                        unsigned long long *d_arrive, bool mc, void *scratch,
                                        size_t scratch_bytes, cudaStream_t st, int num_sms,
                                        int *launches) {
    *launches = 0;
    if (scratch_bytes < consume_scratch_bytes(num_sms)) return cudaErrorInvalidValue;
    GenArgs g = g0;
    g.hist_only = d_pow == nullptr ? 1u : 0u;
    g.out = d_out;
    scratch_layout(g, scratch, num_sms);
    const uint64_t tasks = (g.n_streams + 31u) / 32u;
    int grid = num_sms;
    if ((uint64_t)grid > tasks) grid = (int)tasks;
    if (grid < 1) grid = 1;
    const MrgKind k = mrg_kind(g, alg1);
    const bool w = d_out != nullptr;
    cudaError_t e;
    if (alg1)
        e = k.specb ? (k.eq4 ? cons_mrg_launch<true, true, true, true>(g, w, grid, st)
                             : cons_mrg_launch<false, true, true, true>(g, w, grid, st))
                    : (k.eq4 ? cons_mrg_launch<true, false, true, false>(g, w, grid, st)
                             : cons_mrg_launch<false, false, true, false>(g, w, grid, st));
    else if (k.specb)
        e = k.eq4 ? (k.samew ? cons_mrg_launch<true, true, false, true>(g, w, grid, st)
                             : cons_mrg_launch<true, false, false, true>(g, w, grid, st))
                  : (k.samew ? cons_mrg_launch<false, true, false, true>(g, w, grid, st)
                             : cons_mrg_launch<false, false, false, true>(g, w, grid, st));
    else
        e = k.eq4 ? (k.samew ? cons_mrg_launch<true, true, false, false>(g, w, grid, st)
                             : cons_mrg_launch<true, false, false, false>(g, w, grid, st))
                  : (k.samew ? cons_mrg_launch<false, true, false, false>(g, w, grid, st)
                             : cons_mrg_launch<false, false, false, false>(g, w, grid, st));
    if (e != cudaSuccess) return e;
    *launches = 2;
    finalize_launch(mc, st, g.hist_slab, grid, g.hist_spill, g.pow_slab, d_hist,
                                         d_pow, d_count, g.overflow, g.overflow + 1, d_arrive);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches = 3;
    return cudaSuccess;
}

cudaError_t launch_generate_mrg(const GenArgs &g, bool alg1, cudaStream_t st) {
    const size_t smem = kMrgRingBytes + kMrgStageBytes + (size_t)32 * kMrgRingBytes;
    const uint64_t grid = (g.n_streams + 31) / 32;
    if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const MrgKind mk = mrg_kind(g, alg1);
    const bool eq4 = mk.eq4, samew = mk.samew, specb = mk.specb;
    auto k = alg1 ? (specb ? (eq4 ? gen_mrg_kernel<true, true, true, true>
                                  : gen_mrg_kernel<false, true, true, true>)
                           : (eq4 ? gen_mrg_kernel<true, false, true> : gen_mrg_kernel<false, false, true>))
             : specb ? (eq4 ? (samew ? gen_mrg_kernel<true, true, false, true>
                                     : gen_mrg_kernel<true, false, false, true>)
                            : (samew ? gen_mrg_kernel<false, true, false, true>
                                     : gen_mrg_kernel<false, false, false, true>))
                     : eq4 ? (samew ? gen_mrg_kernel<true, true, false> : gen_mrg_kernel<true, false, false>)
                           : (samew ? gen_mrg_kernel<false, true, false>
                                    : gen_mrg_kernel<false, false, false>);
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)grid, 32, smem, st>>>(g);
    return cudaGetLastError();
}

// Eq.(4) with w = 8 or 16 and both draws at full width: the byte-permute composition of the
// jump kernel (and, with PRNGD_JUMP_NARROW_V, gen_jump_narrow_kernel)
bool jump_is_narrow(const GenArgs &g) {
    return PRNGD_JUMP_NARROW && kernel_mode(g) == 1 && (g.w == 8 || g.w == 16) &&
           g.sh1 == 32u - g.w && g.sh2 == 32u - g.w;
}
bool jump_uses_narrow_kernel(const GenArgs &g) {
    return PRNGD_JUMP_NARROW_V && jump_is_narrow(g) && g.span == g.span_fast;
}

template <int P>
static cudaError_t jump_launch(const GenArgs &g, cudaStream_t st) {
    const void *tables = nullptr;  // the byte tables with the lane index innermost
    cudaError_t e = jump_tables_interleaved(2u * P, &tables);
    if (e != cudaSuccess) return e;
    const size_t smem = 1024 + (size_t)kJumpWarps * jump_comp_bytes<P>();
    const uint64_t grid = (g.n_streams + kJumpWarps - 1) / kJumpWarps;
    if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const uint4 *t = static_cast<const uint4 *>(tables);
    const int mode = kernel_mode(g);
#define PRNGD_JUMP_LAUNCH(M)                                                                    \
    do {                                                                                        \
        if ((e = set_smem(gen_jump_kernel<M, P>, smem)) != cudaSuccess) return e;               \
        gen_jump_kernel<M, P><<<(unsigned)grid, kJumpWarps * 32, smem, st>>>(g, t);            \
    } while (0)
    const bool narrow = jump_is_narrow(g);
    switch (mode) {
        case 3: PRNGD_JUMP_LAUNCH(3); break;
        case 2: PRNGD_JUMP_LAUNCH(2); break;
        case 1:
#if PRNGD_JUMP_NARROW_V
            // (Eq.(4) is exact for w <= 26, so the R11 clamp is never needed here: the host's
            // span_fast == span; the check keeps the kernel honest if that ever changed)
            if (jump_uses_narrow_kernel(g)) {
                const size_t sn = 16 + (size_t)kJumpWarps * jumpn_comp_bytes<P>();
                auto kn = g.w == 8 ? gen_jump_narrow_kernel<true, false, P>
                                   : gen_jump_narrow_kernel<false, false, P>;
                if ((e = set_smem(kn, sn)) != cudaSuccess) return e;
                kn<<<(unsigned)grid, kJumpWarps * 32, sn, st>>>(g, t);
                break;
            }
#endif
            if (narrow && g.w == 8) PRNGD_JUMP_LAUNCH(kJumpMode8);
            else if (narrow && g.w == 16) PRNGD_JUMP_LAUNCH(kJumpMode16);
            else PRNGD_JUMP_LAUNCH(1);
            break;
        default: PRNGD_JUMP_LAUNCH(0); break;
    }
#undef PRNGD_JUMP_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_generate_jump(const GenArgs &g, const Plan &pl, cudaStream_t st) {
    (void)pl;
    // long rows: one 33-pair round per 1024 outputs; short rows: 17-pair rounds
    return g.nps >= PRNGD_JUMP_LONG_MIN ? jump_launch<kJumpPairsLong>(g, st)
                                        : jump_launch<kJumpPairs>(g, st);
}

cudaError_t launch_generate_seg(const GenArgs &g, const Plan &pl, cudaStream_t st) {
    const void *tables = nullptr;
    const uint32_t SO = pl.seg_out ? pl.seg_out : (uint32_t)kSegOut;
    const uint64_t S = g.nps / SO;  // host checked: nps = SO * S, S a power of two <= 32
    uint32_t log2S = 0;
    while ((1ull << log2S) < S) ++log2S;
    const uint64_t rows_per_warp = 32u >> log2S;
    const uint64_t n_tasks = (g.n_streams + rows_per_warp - 1) / rows_per_warp;
    const uint32_t F = SO < (uint32_t)kSegHalf ? SO : (uint32_t)kSegHalf;
    const size_t smem = 1024 + (size_t)32 * (F * 8 + 16);
    cudaError_t e;
#if PRNGD_SEG_JUMP == 1 || PRNGD_SEG_JUMP == 2
    if ((e = jump_tables_nibble(2 * SO, &tables)) != cudaSuccess) return e;
#elif PRNGD_SEG_JUMP == 4
    if ((e = jump_tables_interleaved(2 * SO, &tables)) != cudaSuccess) return e;
#else
    if ((e = jump_tables(2 * SO, &tables)) != cudaSuccess) return e;
#endif
    const uint4 *t = static_cast<const uint4 *>(tables);
    const int mode = kernel_mode(g);
    // consecutive tasks per CTA (hides all but the first jump); one when the grid is small
#ifndef PRNGD_SEG_TPC
#define PRNGD_SEG_TPC 4
#endif
    const uint32_t tpc = n_tasks >= 148ull * 12 * 16 ? PRNGD_SEG_TPC : 1u;
    const uint64_t grid = (n_tasks + tpc - 1) / tpc;
    if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
#define PRNGD_SEG_LAUNCH3(M, I, SOV)                                                            \
    do {                                                                                        \
        if ((e = set_smem(gen_seg_kernel<M, I, SOV>, smem)) != cudaSuccess) return e;           \
        gen_seg_kernel<M, I, SOV><<<(unsigned)grid, 32, smem, st>>>(g, t, log2S, n_tasks, tpc); \
    } while (0)
#define PRNGD_SEG_LAUNCH(M, I)                                                                  \
    do {                                                                                        \
        if (SO == 32) PRNGD_SEG_LAUNCH3(M, I, 32);                                              \
        else if (SO == 64) PRNGD_SEG_LAUNCH3(M, I, 64);                                         \
        else PRNGD_SEG_LAUNCH3(M, I, 128);                                                      \
    } while (0)
    if (pl.ieee_div) {
        switch (mode) {
            case 3: case 2: PRNGD_SEG_LAUNCH(3, true); break;
            case 1: PRNGD_SEG_LAUNCH(1, true); break;
            default: PRNGD_SEG_LAUNCH(0, true); break;
        }
    } else {
        switch (mode) {
            case 3: PRNGD_SEG_LAUNCH(3, false); break;
            case 2: PRNGD_SEG_LAUNCH(2, false); break;
            case 1: PRNGD_SEG_LAUNCH(1, false); break;
            default: PRNGD_SEG_LAUNCH(0, false); break;
        }
    }
#undef PRNGD_SEG_LAUNCH
#undef PRNGD_SEG_LAUNCH3
    return cudaGetLastError();
}

cudaError_t launch_generate_segc(const GenArgs &g, const Plan &pl, cudaStream_t st) {
#if !PRNGD_AB_STORES
    (void)g, (void)pl, (void)st;
    return cudaErrorNotSupported;  // A/B variant build only
#else
    // host checked: nps % (8 * 64) == 0, 16-byte aligned output, speculative, pair-drop
    const uint64_t L = g.nps / kSegcWarps;
    const void *tables = nullptr;
    cudaError_t e = jump_tables_nibble(2 * L, &tables);
    if (e != cudaSuccess) return e;
    const uint4 *t = static_cast<const uint4 *>(tables);
    const uint64_t n_tasks = (g.n_streams + 31) / 32;
    const size_t smem = 1024 + (size_t)kSegcTabBytes + (size_t)kSegcWarps * 32 * kSegRS;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t grid = n_tasks < (uint64_t)sms ? n_tasks : (uint64_t)sms;  // one CTA per SM
    const int mode = kernel_mode(g);
#define PRNGD_SEGC_LAUNCH(M, I)                                                                 \
    do {                                                                                        \
        if ((e = set_smem(gen_segc_kernel<M, I>, smem)) != cudaSuccess) return e;               \
        gen_segc_kernel<M, I><<<(unsigned)grid, kSegcWarps * 32, smem, st>>>(g, t, n_tasks);   \
    } while (0)
    if (pl.ieee_div) {
        switch (mode) {
            case 3: case 2: PRNGD_SEGC_LAUNCH(3, true); break;
            case 1: PRNGD_SEGC_LAUNCH(1, true); break;
            default: PRNGD_SEGC_LAUNCH(0, true); break;
        }
    } else {
        switch (mode) {
            case 3: PRNGD_SEGC_LAUNCH(3, false); break;
            case 2: PRNGD_SEGC_LAUNCH(2, false); break;
            case 1: PRNGD_SEGC_LAUNCH(1, false); break;
            default: PRNGD_SEGC_LAUNCH(0, false); break;
        }
    }
#undef PRNGD_SEGC_LAUNCH
    return cudaGetLastError();
#endif
}

cudaError_t launch_debug_raw(const GenArgs &g, uint32_t *d_raw, uint64_t draws, cudaStream_t st) {
    const uint64_t blocks = (g.n_streams + 127) / 128;
    debug_raw_kernel<<<(unsigned)blocks, 128, 0, st>>>(g, d_raw, draws);
    return cudaGetLastError();
}

cudaError_t launch_debug_pairs(const GenArgs &g, const Plan &pl, uint32_t *d_pidx,
                               uint64_t *d_consumed, cudaStream_t st) {
    const uint64_t blocks = (g.n_streams + 127) / 128;
    if (pl.alg1)
        debug_pairs_kernel<true><<<(unsigned)blocks, 128, 0, st>>>(g, d_pidx, d_consumed);
    else
        debug_pairs_kernel<false><<<(unsigned)blocks, 128, 0, st>>>(g, d_pidx, d_consumed);
    return cudaGetLastError();
}

cudaError_t launch_debug_map(const GenArgs &g, const Plan &pl, const uint32_t *x1,
                             const uint32_t *x2, double *z, uint64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (pl.ieee_div)
        debug_map_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(g, x1, x2, z, n);
    else
        debug_map_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(g, x1, x2, z, n);
    return cudaGetLastError();
}

cudaError_t launch_debug_div_check(const GenArgs &g, uint64_t n, uint64_t seed,
                                   unsigned long long *mismatch, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    debug_div_check_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, n, seed, mismatch);
    return cudaGetLastError();
}

}  // namespace prngd
