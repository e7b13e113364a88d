/*
 * prngd.h -- C ABI of the B200-native PRNGD library (libprngd_b200.so).
 *
 * Method: Demchik & Gulov, "Increasing precision of uniform pseudorandom number generators"
 * (arXiv 1401.8230).  Citations are PAPER.md lines ("P:57") and equation numbers; the readings
 * R1..R17 of the paper are listed in DESIGN.md section 2.
 *
 * One output z' is built from one ACCEPTED pair (x1, x2) of w-bit pseudorandom integers:
 *   Eq.(1)  z  = x1 + k*x2,  k = 2^-w
 *   rule    drop the pair if x1 = a0 or x1 = a (more generally unless a0 < x1 < a) (R3)
 *   Eq.(4)  z' = (z - (a0 + k*b)) / (a - a0 - k*(b - b0))  in [0,1)
 * PRNGD(k, min, max) of Alg. 1 is w = -log2(k), a0 = b0 = min, a = b = max.
 *
 * The base generator is Marsaglia's xorshift128 (one per "stream"), seeded per stream from
 * SplitMix64(seed) (R6).  x1 and x2 are the top bitlen(a) / bitlen(b) bits of consecutive
 * draws (R4).  Output j of stream s is produced by the j-th accepted pair of that stream (R2),
 * so every stream yields exactly n_per_stream outputs and the layout is deterministic.
 *
 * Conventions for every entry point:
 *   - Device pointers ("d_") are CUDA device memory on the current device, owned by the caller.
 *     Host pointers ("h_") are host memory owned by the caller (pinned memory is fastest).
 *   - Work is enqueued on `cuda_stream` (a cudaStream_t; NULL = the legacy default stream) and
 *     the call returns without synchronising, except prngd_generate_host which returns after
 *     the host buffer is complete.  Kernel faults surface at the caller's next synchronisation.
 *   - No call throws or aborts; errors are returned as prngd_status, with a detail string in
 *     prngd_last_error() (thread-local).  A handle is immutable after prngd_create, so several
 *     threads may use one handle concurrently on different streams / buffers -- with one
 *     exception: prngd_generate_consume reduces through per-handle device scratch (per-SM
 *     histogram slabs, carry array, overflow flag), so its calls on ONE handle must be ordered
 *     on one stream; concurrent consumers use separate handles.
 */
#ifndef PRNGD_H
#define PRNGD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRNGD_ABI_VERSION 1

#if defined(__GNUC__)
#define PRNGD_API __attribute__((visibility("default")))
#else
#define PRNGD_API
#endif

typedef enum {
    PRNGD_OK = 0,
    PRNGD_EINVAL = 1,       /* invalid parameters, NULL or misaligned pointer, size overflow */
    PRNGD_ECUDA = 2,        /* a CUDA runtime / driver call or a kernel launch failed */
    PRNGD_ENOMEM = 3,       /* device or host allocation failed */
    PRNGD_EUNSUPPORTED = 4  /* no sm_100a device, or a flag combination not implemented */
} prngd_status;

/* flags */
#define PRNGD_FLAG_IEEE_DIV   0x1u  /* use the IEEE division instruction sequence instead of the
                                       reciprocal + 2 FMA correction (R10); same bits, slower */
/* Store-path selection, bits 3..5 (every path writes the same bits).  The product library
 * implements AUTO, ROW and SEG; TMA, TILE, DIRECT, ROW1K and SEGC were measured slower
 * and exist only in the A/B variant build (-DPRNGD_AB_STORES=1,
 * tools/ab_variants.sh): the product library returns PRNGD_EUNSUPPORTED for them.
 *   AUTO   (default, 0) ROW for bulk shapes; for few streams (n_streams < 16384, n_per_stream
 *          >= 512) SEG when rejection is rare, else the NEXT-3 jump kernel; the fused consumer
 *          always stages ROW tiles beside its histogram
 *   SEG    row segments: n_per_stream / 128 lanes share a row, lane j starts at pair 128 j of
 *          its stream by GF(2) jump-ahead and owns that 1 KiB segment; each flush writes 512-byte
 *          chunks of every segment.  Needs rare rejection (prngd_info.speculative), pair-drop
 *          consumption and n_per_stream = 128 * 2^m <= 4096; otherwise ROW is used
 *   SEGC   column blocks: a CTA of 8 warps owns 32 rows and warp j writes column block j
 *          (n_per_stream / 8 outputs) of each, its lanes starting at pair j * n_per_stream / 8
 *          by jump-ahead (shared-memory nibble tables); needs rare rejection, pair-drop and
 *          n_per_stream % 512 == 0, otherwise ROW is used
 *   ROW    each warp stages 32 rows x 64 outputs in shared memory and writes every row
 *          as one 512-byte burst (32 lanes x 16-byte st.global) -- DRAM-friendly row bursts
 *   TMA    32 x 16-output warp tiles, one cp.async.bulk.tensor.2d store per 128-row CTA slab
 *   TILE   32 x 16-output warp tiles written with warp-coalesced 16-byte st.global
 *   DIRECT every lane writes its own row from registers with 32-byte st.global.v4
 * A path whose alignment rules the output pointer / n_per_stream break falls back to the next
 * legal one (ROW, TMA, TILE: 16-byte aligned output and even n_per_stream; DIRECT: 32-byte and
 * n_per_stream % 4 == 0; otherwise 8-byte stores). */
#define PRNGD_STORE_SHIFT        3
#define PRNGD_STORE_MASK         (7u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_AUTO    (0u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_ROW     (5u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_SEG     (6u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_SEGC    (7u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_TMA     (1u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_TILE    (2u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_DIRECT  (3u << PRNGD_STORE_SHIFT)
#define PRNGD_FLAG_STORE_ROW1K   (4u << PRNGD_STORE_SHIFT)  /* ROW with 1 KiB bursts (A/B) */
/* Mapping selection, bits 6..7 (NEXT-1): Eq.(4) (default), Eq.(5) discrete-grid normalisation
 * onto [0; 1-k'], or Eq.(6) unit-interval form (requires a0 = b0 = 0 and
 * a = b = 2^w - 1).  All three are followed by the R11 clamp (z' <= 1 - 2^-53). */
#define PRNGD_MAP_SHIFT          6
#define PRNGD_MAP_MASK           (3u << PRNGD_MAP_SHIFT)
#define PRNGD_FLAG_MAP_EQ4       (0u << PRNGD_MAP_SHIFT)
#define PRNGD_FLAG_MAP_EQ5       (1u << PRNGD_MAP_SHIFT)
#define PRNGD_FLAG_MAP_EQ6       (2u << PRNGD_MAP_SHIFT)
#define PRNGD_FLAG_OPEN          0x100u  /* return 1 - z': never 0; the histogram puts
                                            1.0 in bin 65535 (R18) */
/* NEXT-3 intra-stream parallelism: one warp per stream, lanes start at draws 0, 2P, 4P, ... of
 * the stream via GF(2) jump-ahead of xorshift128 (P = 33 pairs per lane for rows of >= 1000
 * outputs, else 17) and a warp scan of accepted counts places every output exactly where the
 * sequential order puts it.  Chosen automatically by prngd_generate
 * when there are too few streams to fill the GPU (AUTO store path, n_streams < 16384 and n_per_stream >= 512,
 * pair-drop consumption); these flags force it on or off. */
/* NEXT-2: MRG32k3a base generator (L'Ecuyer 1999; P:165 names it) instead of xorshift128.
 * x1 and x2 are uniform bitlen(a)- and bitlen(b)-bit values obtained from MRG32k3a outputs by
 * reduce-to-width rejection (both widths <= 31); each stream's state comes from SplitMix64
 * outputs #3s..#3s+2.  Pair-drop, or Alg. 1 with PRNGD_FLAG_ALG1 (an out-of-band x1 is
 * redrawn alone); needs a 16-byte aligned output and even n_per_stream.
 * prngd_generate, prngd_generate_host, and prngd_generate_consume, whose statistics are fused
 * into the generator kernel as on xorshift128 (3 launches: generate + bin, exact pass, slab
 * reduction; outputs optional).  EUNSUPPORTED for the debug hooks and with PRNGD_FLAG_JUMP. */
#define PRNGD_FLAG_MRG32K3A      0x800u
/* prngd_generate_consume counts into per-SM 16-bit packed shared-memory counters.  By default the
 * adds are optimistic (no return value, no carry tracking): each CTA checks afterwards that its
 * counters sum to the outputs it counted, and on a mismatch (a counter wrapped) an exact pass
 * with carry tracking recomputes the histogram in the same call (3 launches per call: consume,
 * exact pass -- which returns at once when nothing wrapped -- and finalize).  This flag uses the
 * carry-tracking adds from the start (2 launches). */
#define PRNGD_FLAG_EXACT_HIST    0x1000u
#define PRNGD_FLAG_JUMP          0x200u
#define PRNGD_FLAG_NO_JUMP       0x400u
#define PRNGD_FLAG_ALG1       0x4u  /* NEXT-2 reading of Alg. 1: a rejected x1 is
                                       redrawn alone (x2 is drawn only after acceptance) */

typedef struct {
    uint32_t w;             /* k = 2^-w, 1 <= w <= 32                                        */
    uint32_t flags;         /* PRNGD_FLAG_*; 0 = canonical (pair-drop, Eq.(4), clamp)         */
    uint64_t a0, a;         /* x1 range [a0; a]: a < 2^32, a - a0 >= 2, and the accept band   */
                            /* a0 < x1 < a holds >= 2^-16 of the 2^bitlen(a) draw values     */
    uint64_t b0, b;         /* x2 range [b0; b]: b0 == 0, b + 1 a power of two, b < 2^w (R5) */
    uint64_t seed;          /* SplitMix64 seed (R6)                                           */
    uint64_t stream_begin;  /* first GLOBAL stream id of this call (multi-GPU shard);         */
                            /* stream_begin + n_streams - 1 <= 2^64 - 1                      */
    uint64_t n_streams;     /* >= 1                                                           */
    uint64_t n_per_stream;  /* >= 1; n_streams * n_per_stream < 2^62; n_per_stream < 2^32     */
} prngd_params;

typedef struct prngd_handle prngd_handle;

typedef struct {
    /* Eq.(3)/(4) constants as the library computed them (R7) and their scaled GPU forms (R10) */
    double C, D;            /* C = a0 + k*b, D = (a - a0) - k*(b - b0)                       */
    double C_s, D_s, y;     /* C*2^w, D*2^w, RN(1/D_s)                                        */
    uint32_t sh1, sh2;      /* x1 = u1 >> sh1, x2 = u2 >> sh2 (R4)                           */
    uint32_t clamp;         /* 1 if some accepted pair maps to 1.0 before the clamp (R11)    */
    uint32_t speculative;   /* 1 if the kernel checks acceptance once per batch (rare rejection) */
    uint64_t n_outputs;     /* n_streams * n_per_stream                                      */
    uint64_t out_bytes;     /* 8 * n_outputs                                                 */
    uint32_t kernel;        /* kernel prngd_generate launches for a 256-byte aligned output:
                               0 gen_kernel (one lane per stream), 1 gen_seg_kernel (SEG),
                               2 gen_jump_kernel (NEXT-3), 3 gen_mrg_kernel (NEXT-2),
                               4 gen_segc_kernel (SEGC), 5 gen_jump_narrow_kernel (NEXT-3,
                               w = 8 / 16 with both draws at full width)                       */
    uint32_t store;         /* its store path: 0 TMA, 1 TILE, 2 8-byte, 3 DIRECT, 4 ROW,
                               5 ROW1K, 6 SEG, 7 SEGC                                         */
} prngd_info;

/* Validate *p and build an immutable handle (host only: no CUDA call, no device memory).
 * Returns PRNGD_EINVAL for parameters outside the domain documented on prngd_params. */
PRNGD_API prngd_status prngd_create(const prngd_params *p, prngd_handle **out);

/* Release a handle and any device scratch it owns.  NULL-safe.  Not synchronising: the caller
 * must not destroy a handle while its work is still running on a stream. */
PRNGD_API prngd_status prngd_destroy(prngd_handle *h);

/* Constants and dispatch choices of the handle (host only). */
PRNGD_API prngd_status prngd_get_info(const prngd_handle *h, prngd_info *info);

/* S1-S6: d_out[i * n_per_stream + j] = output j of global stream stream_begin + i.
 * d_out: device, >= n_streams * n_per_stream doubles, 8-byte aligned (a 16-byte aligned output
 * and an even n_per_stream enable the row-burst store paths; see the store flags above).  One
 * kernel launch; prngd_get_info reports which kernel and store path. */
PRNGD_API prngd_status prngd_generate(const prngd_handle *h, double *d_out, void *cuda_stream);

/* S1-S7: as prngd_generate (outputs written only if d_out != NULL), plus the fused consumer:
 *   d_hist[bin] += #{outputs with (uint32)(z' * 65536.0) == bin}    (65536 int64, R16)
 *   d_pow[p-1] += sum z'^p, p = 1..4                                  (4 doubles)
 *   d_count[0] += number of outputs                                  (1 int64)
 * All three accumulate with device atomics, so shards -- including other processes on other
 * GPUs that mapped the same buffer with prngd_ipc_open (peer memory over NVLink) -- may add
 * into one buffer concurrently: the statistics reduction then happens inside this call's own
 * kernels.  d_hist, d_count: device (local or peer-mapped), 8-byte aligned, required.  d_pow: the
 * same, or NULL for a histogram-only call (BASELINE cfg4's "fused 2^16-bin histogram": d_hist and
 * d_count as above, no power sums; the kernel then skips their five FP64 operations per output).
 * Three kernel launches (generate + bin, the exact pass that returns at once unless a 16-bit
 * counter wrapped, slab reduction); two with PRNGD_FLAG_EXACT_HIST. */
PRNGD_API prngd_status prngd_generate_consume(const prngd_handle *h, double *d_out, int64_t *d_hist,
                                    double *d_pow, int64_t *d_count, void *cuda_stream);

/* As prngd_generate_consume, plus a completion signal for accumulators shared across GPUs:
 * d_arrive (device, local or peer-mapped, 8-byte aligned; NULL = no signal) is incremented by
 * one, with a system-scope release, after every statistic of this call has been added.  A
 * reader that observes *d_arrive >= n (acquire; e.g. prngd_wait_arrivals) sees the complete
 * statistics of those n calls.  The increment happens inside the call's last (finalize) kernel. */
PRNGD_API prngd_status prngd_generate_consume_ex(const prngd_handle *h, double *d_out,
                                                 int64_t *d_hist, double *d_pow, int64_t *d_count,
                                                 uint64_t *d_arrive, void *cuda_stream);

/* Enqueue on cuda_stream a one-thread kernel that waits (system-scope acquire loads) until
 * *d_arrive >= target; later work on the stream then sees every add those arrivals covered.
 * For ranks on DIFFERENT GPUs (a rank waiting on kernels of another process on the same GPU
 * can starve them).  timeout_ns (0 = 60 s) bounds the wait: on expiry the kernel traps, which
 * the caller sees as a launch failure at its next synchronisation. */
PRNGD_API prngd_status prngd_wait_arrivals(const uint64_t *d_arrive, uint64_t target,
                                           uint64_t timeout_ns, void *cuda_stream);

/* End-to-end form for host memory: h_out (host, >= n_outputs doubles) receives the same
 * values as prngd_generate would write.  Generates in chunks of streams into device scratch
 * owned by the handle and overlaps the device->host copies with generation.  Synchronous:
 * returns after h_out is complete.  PRNGD_ENOMEM if the scratch cannot be allocated. */
PRNGD_API prngd_status prngd_generate_host(prngd_handle *h, double *h_out, void *cuda_stream);

/* Number of kernel launches the last successful call on this handle enqueued. */
PRNGD_API uint32_t prngd_last_launches(const prngd_handle *h);

PRNGD_API const char *prngd_status_string(prngd_status s);
PRNGD_API const char *prngd_last_error(void);
PRNGD_API int prngd_abi_version(void);

/* ---- validation hooks (not timed; same __device__ code as the production kernels) ---- */

/* d_raw[i * draws_per_stream + d] = d-th xorshift128 output of global stream stream_begin+i. */
PRNGD_API prngd_status prngd_debug_raw(const prngd_handle *h, uint32_t *d_raw, uint64_t draws_per_stream,
                             void *cuda_stream);

/* d_pair_index[i * n_per_stream + j] = 0-based index of the pair that produced output j of
 * stream i (pair p = draws 2p, 2p+1), modulo 2^32; d_pairs_consumed[i] = pairs consumed by
 * stream i (64-bit).  Either pointer may be NULL. */
PRNGD_API prngd_status prngd_debug_pairs(const prngd_handle *h, uint32_t *d_pair_index,
                               uint64_t *d_pairs_consumed, void *cuda_stream);

/* d_z[i] = Eq.(4) + clamp of the pair (d_x1[i], d_x2[i]) in integer units, through the same
 * device mapping as the generator (no acceptance test).  n may be 0. */
PRNGD_API prngd_status prngd_debug_map(const prngd_handle *h, const uint32_t *d_x1, const uint32_t *d_x2,
                             double *d_z, uint64_t n, void *cuda_stream);

/* Host-only check of the jump-ahead: out = T^n_draws * in for the xorshift128 state
 * (x, y, z, w) = in[0..3].  lane_table >= 0 applies instead the byte table the GPU uses for lane
 * `lane_table` (= T^(d * lane_table)) with per-lane distance d = n_draws, or d = 34 (the NEXT-3
 * jump kernel's tables) when n_draws is 0; the SEG store path uses d = 256.  No CUDA call. */
PRNGD_API prngd_status prngd_debug_jump(uint64_t n_draws, const uint32_t *in, uint32_t *out,
                                        int lane_table);

/* d_mismatch[0] += number of n_s in the sample for which the reciprocal + 2 FMA quotient
 * differs from the IEEE division (R10).  Samples: n = RN(v) - C_s for v = x1*2^w + x2 with
 * (x1, x2) from a counter-based hash of (seed, i), i < n.  Validation of R10 on the GPU. */
PRNGD_API prngd_status prngd_debug_div_check(const prngd_handle *h, uint64_t n, uint64_t seed,
                                   unsigned long long *d_mismatch, void *cuda_stream);

/* ---- Peer-memory plumbing for the multi-GPU statistics reduction (SURVEY 8(e), NEXT-4 over
 * NVLink peer memory instead of multicast).  One process allocates the accumulator
 * (prngd_peer_alloc: zeroed device memory of this process's current device), exports it
 * (prngd_ipc_export: PRNGD_IPC_HANDLE_BYTES opaque bytes, to be sent to the other processes of
 * the node by any means), and every other process maps it (prngd_ipc_open) and passes the
 * mapped pointers to prngd_generate_consume.  prngd_copy / prngd_zero are stream-ordered
 * device copies / zero-fills of such raw allocations.  All return PRNGD_ECUDA with the CUDA
 * error in prngd_last_error() when the runtime refuses (e.g. no peer access). */
#define PRNGD_IPC_HANDLE_BYTES 64
PRNGD_API prngd_status prngd_peer_alloc(uint64_t bytes, void **d_ptr);
PRNGD_API prngd_status prngd_peer_free(void *d_ptr);
PRNGD_API prngd_status prngd_ipc_export(void *d_ptr, void *handle_out);
PRNGD_API prngd_status prngd_ipc_open(const void *handle, void **d_ptr);
PRNGD_API prngd_status prngd_ipc_close(void *d_ptr);
PRNGD_API prngd_status prngd_copy(void *dst, const void *src, uint64_t bytes, void *cuda_stream);
PRNGD_API prngd_status prngd_zero(void *d_ptr, uint64_t bytes, void *cuda_stream);

/* ---- NEXT-4: NVLS multicast statistics (in-switch all-reduce inside the finalize kernel).
 * Layout of a shared statistics buffer (PeerStats and multicast alike), 8-byte words:
 *   [0, 65536) int64 histogram | count int64 | 4 x double power sums | uint64 arrival counter */
#define PRNGD_STATS_COUNT_OFFSET  (65536u * 8u)
#define PRNGD_STATS_POW_OFFSET    (65537u * 8u)
#define PRNGD_STATS_ARRIVE_OFFSET (65541u * 8u)
#define PRNGD_STATS_BYTES         (65542u * 8u)

/* As prngd_generate_consume_ex with the statistics buffer (layout above) given by its NVLS
 * MULTICAST address (prngd_mc_bind_map's *mc_ptr): the finalize kernel adds the histogram, count
 * and power sums with multimem.red (the NVSwitch performs each add on every member GPU's copy)
 * and then increments the arrival counter with a multimem.red.release -- so after R ranks' calls
 * every rank's LOCAL copy holds the all-reduced statistics and an arrival count of R, with no
 * collective call.  Requires a multicast object bound on every rank (below). */
PRNGD_API prngd_status prngd_generate_consume_mc(const prngd_handle *h, double *d_out,
                                                 void *mc_stats, void *cuda_stream);

/* Multicast accumulator setup, one process per GPU, driven by the caller's process group:
 *   1. owner: prngd_mc_create(bytes, R, &m, &fd); broadcast (getpid(), fd)
 *   2. others: prngd_mc_import(owner_pid, fd, prngd_mc_bytes, &m)  (pidfd_getfd)
 *   3. every rank: prngd_mc_add_device(m); barrier
 *   4. every rank: prngd_mc_bind_map(m, &mc_ptr, &local_ptr) (zeroed local copy); barrier
 *   5. prngd_mc_destroy(m) on every rank (after a barrier) when done.
 * To let the other ranks fetch the descriptor with pidfd_getfd, prngd_mc_create allows ptrace
 * attachment to the owner process (PR_SET_PTRACER_ANY, Yama) until the owner's
 * prngd_mc_bind_map, which withdraws it and closes the exported descriptor.
 * prngd_mc_supported reports CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED for the current device.
 * Any step returns PRNGD_ECUDA / PRNGD_EUNSUPPORTED with the driver's reason when the fabric or
 * the driver cannot provide the object (e.g. one-GPU leases: cuMulticastCreate refuses); callers
 * then fall back to peer memory or NCCL (paper_1401_8230_b200.dist). */
typedef struct prngd_mc prngd_mc;
PRNGD_API prngd_status prngd_mc_supported(int *supported);
PRNGD_API prngd_status prngd_mc_create(uint64_t bytes, uint32_t n_devices, prngd_mc **out,
                                       int *export_fd);
PRNGD_API prngd_status prngd_mc_import(int owner_pid, int owner_fd, uint64_t bytes, prngd_mc **out);
PRNGD_API uint64_t prngd_mc_bytes(const prngd_mc *m);
PRNGD_API prngd_status prngd_mc_add_device(prngd_mc *m);
PRNGD_API prngd_status prngd_mc_bind_map(prngd_mc *m, void **mc_ptr, void **local_ptr);
PRNGD_API prngd_status prngd_mc_destroy(prngd_mc *m);

#ifdef __cplusplus
}
#endif
#endif /* PRNGD_H */
