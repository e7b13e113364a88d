// prngd_internal.h -- structures shared by the host runtime (prngd_host.cpp) and the sm_100a
// kernels (prngd_kernels.cu).  Product code only; nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/prngd.h"

namespace prngd {

// Mapping constants of the generic kernels (prngd_device.cuh map_pair): Eq.(4)/(5)/(6) scaled by
// 2^w (R10) plus the open-interval switch.
struct MapArgs {
    double Cs, Ds, y, scale;
    uint32_t w, sub, kind, open;
};

// Everything a generator kernel needs, by value in the kernel parameter bank.
struct GenArgs {
    uint64_t seed;          // SplitMix64 seed (R6)
    uint64_t stream_begin;  // global id of row 0
    uint64_t n_streams;     // rows
    uint64_t nps;           // n_per_stream, columns
    double *out;            // row-major [n_streams][nps]; may be null in consume-only mode
    double Cs, Ds, y;       // C*2^w, D*2^w, RN(1/D_s)   (R10)
    uint32_t w;             // composition shift, v = (x1 << w) | x2
    uint32_t sh1, sh2;      // draw widths, x = u >> sh (R4)
    uint32_t lo, span;      // accept iff (x1 - lo) < span  <=>  a0 < x1 < a   (R3)
    uint32_t span_fast;     // span - clamp: speculative band excluding x1 = a - 1 when R11 applies
    uint32_t pow2w;         // 2^w for w <= 31 (v = x1 * 2^w + x2 in one wide multiply-add), else 0
    MapArgs map;            // mapping of the generic kernels (Eq.(4)/(5)/(6), open interval)
    uint32_t mrg_t1, mrg_t2;        // NEXT-2: reduce-to-width thresholds for bitlen(a), bitlen(b)
    uint32_t mrg_mask1, mrg_mask2;  //         and the width masks
    double mrg_m1, mrg_inv1, mrg_m2, mrg_inv2;  // MRG32k3a moduli and RN(1/m) (binary64 form)
    // consumer (S7)
    uint32_t *hist_slab;    // [gridDim.x][65536] one u32 per bin (consume kernels only)
    int64_t *hist_spill;    // [65536] int64 carries of the packed counters
    double *pow_slab;       // [gridDim.x][4]
    uint32_t *overflow;     // set by an optimistic (RED) consume kernel whose 16-bit fields wrapped
    // fused consumer with row segments (Store::SEG): log2 of the lanes per row and the
    // lane-interleaved jump tables of distance kSegDraws
    uint32_t seg_log2;
    // histogram-only consumer (the caller passed no power-sum accumulator: BASELINE cfg4's "fused
    // 2^16-bin histogram"): the full-batch fast paths skip the five FP64 power-sum operations
    uint32_t hist_only;
    const uint4 *jump_tab;
};

// How a warp's outputs reach HBM (include/prngd.h PRNGD_FLAG_STORE_*):
//   ROW:    32 rows x 64 outputs staged in smem, each row written as one 512 B burst
//   DIRECT: each lane stores its row segment from registers, 4 x 32-byte st.global.v4.f64
//   TMA:    32 x 16 smem tiles (128B swizzle) + one cp.async.bulk.tensor.2d store per CTA slab
//   STG16:  32 x 16 smem tile + warp-coalesced 16-byte st.global;  STG8: 8-byte stores
//   ROW1K:  as ROW with 128 outputs (1 KiB bursts) per row
//   SEG:    nps/128 lanes per row (jump-ahead), each lane a 1 KiB segment; 512 B bursts
//   SEGC:   a CTA of 8 warps owns 32 rows, warp j column block j (jump-ahead); 512 B bursts
enum class Store : int {
    TMA = 0, STG16 = 1, STG8 = 2, DIRECT = 3, ROW = 4, ROW1K = 5, SEG = 6, SEGC = 7
};

// Store paths measured slower than ROW / SEG (TMA, TILE = STG16, DIRECT, ROW1K, SEGC; DESIGN.md
// section 5) are instantiated only in the A/B variant build (tools/ab_variants.sh passes
// -DPRNGD_AB_STORES=1); the product library rejects their flags with PRNGD_EUNSUPPORTED.
#ifndef PRNGD_AB_STORES
#define PRNGD_AB_STORES 0
#endif

// Launch descriptors chosen by the host.
struct Plan {
    bool spec;      // speculative batch acceptance (rare rejection)
    bool clamp;     // R11 clamp needed
    bool ieee_div;  // PRNGD_FLAG_IEEE_DIV
    bool alg1;      // PRNGD_FLAG_ALG1
    bool jump;      // NEXT-3 intra-stream kernel (one warp per stream)
    bool mrg;       // NEXT-2 MRG32k3a base generator
    bool store_auto;  // PRNGD_FLAG_STORE_AUTO: the library picks the store path / kernel
    bool exact_hist;  // PRNGD_FLAG_EXACT_HIST: carry-tracking histogram adds from the start
    uint32_t seg_out; // SEG: outputs per lane segment (128, or 64 / 32 for few-stream shapes)
    Store store;
};

// NEXT-3 jump-ahead (prngd_jump.cpp): lane l of a warp starts a round at draw l*kJumpDraws of
// its stream (kJumpDraws / 2 = 17 pairs per lane per round, 32 lanes per stream: two rounds
// cover a 1024-output row with up to 5.9% rejection, so no sequential tail is needed); rows of
// >= 1000 outputs use 33-pair rounds instead (prngd_kernels.cu kJumpPairsLong, distance 66).
#ifndef PRNGD_JUMP_PAIRS
#define PRNGD_JUMP_PAIRS 17  // cfg2 A/B: 16 -> 224, 17 -> 249-251, 18 -> 232, 24 -> 224 Gd/s
#endif
constexpr uint64_t kJumpDraws = 2 * PRNGD_JUMP_PAIRS;
// SEG store path: a lane owns a 1 KiB segment (kSegOut outputs = pairs) of its stream's row and
// starts at draw j * kSegDraws (segment j) via the same byte tables built for that distance.
constexpr uint64_t kSegOut = 128;
constexpr uint64_t kSegDraws = 2 * kSegOut;
// device byte tables [32][16][256] x uint4 of J_l = T^(lane_draws * l), cached per device
cudaError_t jump_tables(uint64_t lane_draws, const void **out);
// the same matrices as nibble tables [32][32][16] x uint4 (8 KiB per lane matrix)
cudaError_t jump_tables_nibble(uint64_t lane_draws, const void **out);
// the byte tables with the lane index innermost, [16][256][32] x uint4
cudaError_t jump_tables_interleaved(uint64_t lane_draws, const void **out);
void jump_host(uint64_t n_draws, const uint32_t in[4], uint32_t out[4], int lane_table);

// detail string of prngd_last_error() (thread-local), for the other translation units
void set_last_error(const char *msg);

// Launchers (prngd_kernels.cu).  They return cudaGetLastError() of the launch.
cudaError_t launch_generate(const GenArgs &g, const Plan &pl, cudaStream_t st, int num_sms);
// d_arrive (nullable): +1 with a system-scope release once every statistic of the call is added
// mc: the accumulators are an NVLS multicast address (multimem.red in the finalize kernel)
cudaError_t launch_generate_consume(const GenArgs &g, const Plan &pl, double *d_out,
                                    int64_t *d_hist, double *d_pow, int64_t *d_count,
                                    unsigned long long *d_arrive, bool mc, void *scratch,
                                    size_t scratch_bytes, cudaStream_t st, int num_sms,
                                    int *launches);
size_t consume_scratch_bytes(int num_sms);
// S7 over n values already in device memory (src): histogram kernel, exact pass, finalize
cudaError_t launch_consume_memory(const GenArgs &g, const double *src, uint64_t n, int64_t *d_hist,
                                  double *d_pow, int64_t *d_count, unsigned long long *d_arrive,
                                  void *scratch, size_t scratch_bytes, cudaStream_t st,
                                  int num_sms, int *launches);
cudaError_t launch_wait_arrivals(const unsigned long long *arrive, unsigned long long target,
                                 unsigned long long timeout_ns, cudaStream_t st);
cudaError_t launch_generate_mrg(const GenArgs &g, bool alg1, cudaStream_t st);
// S1-S7 on MRG32k3a fused into the generator (d_out null: statistics only); 3 launches
cudaError_t launch_generate_consume_mrg(const GenArgs &g, bool alg1, double *d_out,
                                        int64_t *d_hist, double *d_pow, int64_t *d_count,
                                        unsigned long long *d_arrive, bool mc, void *scratch,
                                        size_t scratch_bytes, cudaStream_t st, int num_sms,
                                        int *launches);
// the jump / SEG launchers fetch (build once per device) the jump tables they read
cudaError_t launch_generate_jump(const GenArgs &g, const Plan &pl, cudaStream_t st);
bool jump_uses_narrow_kernel(const GenArgs &g);  // the jump plan runs gen_jump_narrow_kernel
cudaError_t launch_generate_seg(const GenArgs &g, const Plan &pl, cudaStream_t st);
cudaError_t launch_generate_segc(const GenArgs &g, const Plan &pl, cudaStream_t st);
cudaError_t launch_debug_raw(const GenArgs &g, uint32_t *d_raw, uint64_t draws, cudaStream_t st);
cudaError_t launch_debug_pairs(const GenArgs &g, const Plan &pl, uint32_t *d_pidx,
                               uint64_t *d_consumed, cudaStream_t st);
cudaError_t launch_debug_map(const GenArgs &g, const Plan &pl, const uint32_t *x1,
                             const uint32_t *x2, double *z, uint64_t n, cudaStream_t st);
cudaError_t launch_debug_div_check(const GenArgs &g, uint64_t n, uint64_t seed,
                                   unsigned long long *mismatch, cudaStream_t st);

}  // namespace prngd
