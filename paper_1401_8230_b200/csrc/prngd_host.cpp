// prngd_host.cpp -- C ABI (include/prngd.h): validation, Eq.(3)/(4) constants, dispatch,
// host-buffer pipeline.  Product code; written independently of oracle/.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include "prngd_internal.h"

using prngd::GenArgs;
using prngd::Plan;
using prngd::Store;

struct prngd_handle {
    prngd_params p;
    prngd_info info;
    GenArgs args;
    Plan plan;
    mutable std::atomic<uint32_t> last_launches{0};
    // device scratch, created lazily (consume slabs, host-pipeline staging)
    std::mutex mu;
    int scratch_dev = -1;
    void *cons_scratch = nullptr;
    size_t cons_bytes = 0;
    double *stage[2] = {nullptr, nullptr};
    size_t stage_rows[2] = {0, 0};
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_gen[2] = {nullptr, nullptr};
    cudaEvent_t ev_copy[2] = {nullptr, nullptr};
    // recorded after the last reader of stage[0] enqueued by the MRG32k3a consume-only path;
    // every later user of the staging buffers waits on it (the calls may use other streams)
    cudaEvent_t ev_stage_free = nullptr;
    bool stage_pending = false;
};

static thread_local char g_err[512] = "";

static prngd_status fail(prngd_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

void prngd::set_last_error(const char *msg) {
    std::snprintf(g_err, sizeof(g_err), "%s", msg);
}

static prngd_status cuda_fail(cudaError_t e, const char *what) {
    return fail(PRNGD_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

static int bit_length(uint64_t v) {
    int n = 0;
    for (; v; v >>= 1) ++n;
    return n;
}

// Device checks done once per (thread, device): sm_100 and SM count.
static prngd_status device_ready(int *num_sms) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int major = 0, minor = 0, sms = 0;
    if ((e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess)
        return cuda_fail(e, "cudaDeviceGetAttribute");
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (major != 10 || minor != 0)
        return fail(PRNGD_EUNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                    dev, major, minor);
    *num_sms = sms;
    return PRNGD_OK;
}

// NVTX ranges around the public calls (SURVEY section 5 "tracing"): free unless a profiler such as
// nsys injects its tool library.
namespace {
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace

extern "C" {

const char *prngd_status_string(prngd_status s) {
    switch (s) {
        case PRNGD_OK: return "PRNGD_OK";
        case PRNGD_EINVAL: return "PRNGD_EINVAL: invalid argument";
        case PRNGD_ECUDA: return "PRNGD_ECUDA: CUDA error";
        case PRNGD_ENOMEM: return "PRNGD_ENOMEM: out of memory";
        case PRNGD_EUNSUPPORTED: return "PRNGD_EUNSUPPORTED: unsupported device or option";
    }
    return "PRNGD_?: unknown status";
}

const char *prngd_last_error(void) { return g_err; }

int prngd_abi_version(void) { return PRNGD_ABI_VERSION; }

prngd_status prngd_create(const prngd_params *p, prngd_handle **out) {
    NvtxRange nvtx_range("prngd_create");
    g_err[0] = 0;
    if (!p || !out) return fail(PRNGD_EINVAL, "null argument");
    *out = nullptr;
    const uint32_t w = p->w;
    if (w < 1 || w > 32) return fail(PRNGD_EINVAL, "w=%u outside [1, 32]", w);
    if (p->a > 0xFFFFFFFFull) return fail(PRNGD_EINVAL, "a=%llu does not fit 32 bits",
                                          (unsigned long long)p->a);
    if (p->a0 >= p->a || p->a - p->a0 < 2)
        return fail(PRNGD_EINVAL, "need a - a0 >= 2 (got a0=%llu, a=%llu): no x1 strictly inside",
                    (unsigned long long)p->a0, (unsigned long long)p->a);
    if (p->b0 != 0) return fail(PRNGD_EINVAL, "b0 must be 0 (x2 fills its draw width, R5)");
    if (p->b == 0 || p->b > 0xFFFFFFFFull || ((p->b + 1) & p->b) != 0)
        return fail(PRNGD_EINVAL, "b + 1 must be a power of two <= 2^32 (R5), got b=%llu",
                    (unsigned long long)p->b);
    if (p->b >= (1ull << w))
        return fail(PRNGD_EINVAL, "need b < 2^w so that k*(b - b0) < 1 (b=%llu, w=%u)",
                    (unsigned long long)p->b, w);
    if (p->n_streams == 0 || p->n_per_stream == 0)
        return fail(PRNGD_EINVAL, "n_streams and n_per_stream must be >= 1");
    if (p->n_per_stream >= (1ull << 32))
        return fail(PRNGD_EINVAL, "n_per_stream must be < 2^32");
    if (p->n_streams > (1ull << 62) / p->n_per_stream)
        return fail(PRNGD_EINVAL, "n_streams * n_per_stream overflows (limit 2^62)");
    if (p->n_streams - 1 > ~0ull - p->stream_begin)  // the last stream id must fit 64 bits
        return fail(PRNGD_EINVAL, "stream_begin + n_streams - 1 overflows 64 bits");
    const uint32_t known = PRNGD_FLAG_IEEE_DIV | PRNGD_FLAG_ALG1 | PRNGD_STORE_MASK |
                           PRNGD_MAP_MASK | PRNGD_FLAG_OPEN | PRNGD_FLAG_JUMP | PRNGD_FLAG_NO_JUMP |
                           PRNGD_FLAG_MRG32K3A | PRNGD_FLAG_EXACT_HIST;
    const bool mrg = (p->flags & PRNGD_FLAG_MRG32K3A) != 0;
    if (mrg && (bit_length(p->a) > 31 || bit_length(p->b) > 31))
        return fail(PRNGD_EINVAL, "MRG32k3a draws are at most 31 bits wide (bitlen(a), bitlen(b) <= 31)");
    if (mrg && (p->flags & PRNGD_FLAG_JUMP))
        return fail(PRNGD_EUNSUPPORTED, "MRG32k3a has no jump-ahead path");
    if ((p->flags & PRNGD_FLAG_JUMP) && (p->flags & (PRNGD_FLAG_NO_JUMP | PRNGD_FLAG_ALG1)))
        return fail(PRNGD_EUNSUPPORTED, "jump-ahead needs pair-drop consumption and no NO_JUMP");
    if (p->flags & ~known) return fail(PRNGD_EUNSUPPORTED, "unknown flag bits 0x%x", p->flags & ~known);
    const uint32_t map_code = (p->flags & PRNGD_MAP_MASK) >> PRNGD_MAP_SHIFT;
    if (map_code > 2) return fail(PRNGD_EUNSUPPORTED, "unknown mapping code %u", map_code);
    if (map_code == 2 && !(p->a0 == 0 && p->b0 == 0 && p->a == (1ull << w) - 1 && p->b == p->a))
        return fail(PRNGD_EINVAL, "Eq.(6) needs the unit-interval range a0=b0=0, a=b=2^w-1");
    if (((p->flags & PRNGD_STORE_MASK) >> PRNGD_STORE_SHIFT) > 7)
        return fail(PRNGD_EUNSUPPORTED, "unknown store path %u",
                    (p->flags & PRNGD_STORE_MASK) >> PRNGD_STORE_SHIFT);
#if !PRNGD_AB_STORES
    {
        const uint32_t sp = p->flags & PRNGD_STORE_MASK;
        if (sp != PRNGD_FLAG_STORE_AUTO && sp != PRNGD_FLAG_STORE_ROW && sp != PRNGD_FLAG_STORE_SEG)
            return fail(PRNGD_EUNSUPPORTED,
                        "store path %u is an A/B path of the variant build (-DPRNGD_AB_STORES=1); "
                        "the product library has AUTO, ROW and SEG", sp >> PRNGD_STORE_SHIFT);
    }
#endif
    // Accept band bound: one output costs 2^bitlen(a) / (a - a0 - 1) pairs on average; bands
    // accepting fewer than 2^-16 of the x1 draws are refused (a near-empty band would stall a
    // stream for ~2^31 pairs and wrap the 32-bit pair indices of prngd_debug_pairs).
    if ((p->a - p->a0 - 1) << 16 < (1ull << bit_length(p->a)))
        return fail(PRNGD_EINVAL,
                    "accept band a0 < x1 < a holds %llu of 2^%d draw values: below the 2^-16 "
                    "acceptance floor", (unsigned long long)(p->a - p->a0 - 1), bit_length(p->a));

    prngd_handle *h = new (std::nothrow) prngd_handle();
    if (!h) return fail(PRNGD_ENOMEM, "host allocation of the handle failed");
    h->p = *p;

    // Eq.(3)/(4) constants in IEEE binary64 round-to-nearest, one rounding per operation (R7).
    const double k = std::ldexp(1.0, -(int)w);
    volatile double kb = k * (double)p->b;            // volatile: no contraction / reassociation
    const double C = (double)p->a0 + kb;               // a0 + k*b          (Eq.(3))
    volatile double kbb = k * ((double)p->b - (double)p->b0);
    const double D = ((double)p->a - (double)p->a0) - kbb;  // a - a0 - k(b-b0) (Eq.(4))
    prngd_info &I = h->info;
    I.C = C;
    I.D = D;
    I.C_s = std::ldexp(C, (int)w);                     // exact power-of-two scaling (R10)
    I.D_s = std::ldexp(D, (int)w);
    I.y = 1.0 / I.D_s;                                 // RN(1/D_s)
    I.sh1 = 32u - (uint32_t)bit_length(p->a);
    I.sh2 = 32u - (uint32_t)bit_length(p->b);

    // Mapping constants (scaled by 2^w, R10) for Eq.(4), Eq.(5) or Eq.(6).
    const uint32_t kind = map_code == 1 ? 5u : (map_code == 2 ? 6u : 4u);
    volatile double kk = k * k;                          // k' = k^2 (exact)
    const double scale = 1.0 - kk;                       // RN(1 - k')
    double Ds = I.D_s, Cs = I.C_s;
    uint32_t sub = 0;
    if (kind == 5) {  // den = trunc[(a-a0-2k)/k] + b - b0, in units of k
        volatile double kb5 = k * ((double)p->b - (double)p->b0);
        const double den = (double)(p->a - p->a0 - 2) + kb5;
        Ds = std::ldexp(den, (int)w);
        Cs = 0.0;
        sub = (uint32_t)(p->a0 + 1);
    } else if (kind == 6) {  // den = trunc[1/k] - 2 - k
        volatile double d1 = std::ldexp(1.0, (int)w) - 2.0;
        const double den = d1 - k;
        Ds = std::ldexp(den, (int)w);
        Cs = std::ldexp(1.0, (int)w);                    // the "- 1" of Eq.(6), scaled
    }
    const double y = 1.0 / Ds;                           // RN(1/D_s)
    if (kind == 4) I.y = y;
    // R11: every mapping is monotone, so the largest accepted pair (a-1, b) bounds every output.
    {
        const uint64_t v = ((p->a - 1 - sub) << w) | p->b;
        volatile double n = (double)v - Cs;
        if (kind == 6) n = n * scale;
        volatile double qmax = n / Ds;
        if (kind == 5) qmax = qmax * scale;
        I.clamp = qmax >= 1.0 ? 1u : 0u;
    }
    // Rejection probability per attempt: (draw values outside (a0, a)) / 2^bitlen(a).
    const double width = std::ldexp(1.0, bit_length(p->a));
    const double p_rej = (width - (double)(p->a - p->a0 - 1)) / width;
    // Speculate when a 512-pair warp batch is rejection-free with probability > 99%.
    const bool alg1 = (p->flags & PRNGD_FLAG_ALG1) != 0;
    I.speculative = (!alg1 && p_rej * 512.0 < 0.01) ? 1u : 0u;
    I.n_outputs = p->n_streams * p->n_per_stream;
    I.out_bytes = I.n_outputs * 8u;

    GenArgs &g = h->args;
    std::memset(&g, 0, sizeof(g));
    g.seed = p->seed;
    g.stream_begin = p->stream_begin;
    g.n_streams = p->n_streams;
    g.nps = p->n_per_stream;
    g.Cs = I.C_s;
    g.Ds = I.D_s;
    g.y = I.y;
    g.w = w;
    g.sh1 = I.sh1;
    g.sh2 = I.sh2;
    g.lo = (uint32_t)(p->a0 + 1);
    g.span = (uint32_t)(p->a - p->a0 - 1);
    g.span_fast = g.span - I.clamp;
    g.pow2w = w < 32 ? (1u << w) : 0u;
    g.map.Cs = Cs;
    g.map.Ds = Ds;
    g.map.y = y;
    g.map.scale = scale;
    g.map.w = w;
    g.map.sub = sub;
    g.map.kind = kind;
    g.map.open = (p->flags & PRNGD_FLAG_OPEN) ? 1u : 0u;

    Plan &pl = h->plan;
    pl.spec = I.speculative != 0;
    pl.clamp = I.clamp != 0;
    pl.ieee_div = (p->flags & PRNGD_FLAG_IEEE_DIV) != 0;
    pl.alg1 = alg1;
    pl.mrg = mrg;
    if (mrg) {  // R23 thresholds: T = floor(m1 / 2^width) * 2^width
        const uint64_t m1 = 4294967087ull;
        const uint64_t s1 = 1ull << bit_length(p->a), s2 = 1ull << bit_length(p->b);
        g.mrg_t1 = (uint32_t)(m1 / s1 * s1);
        g.mrg_t2 = (uint32_t)(m1 / s2 * s2);
        g.mrg_mask1 = (uint32_t)(s1 - 1);
        g.mrg_mask2 = (uint32_t)(s2 - 1);
        g.mrg_m1 = 4294967087.0;
        g.mrg_inv1 = 1.0 / 4294967087.0;
        g.mrg_m2 = 4294944443.0;
        g.mrg_inv2 = 1.0 / 4294944443.0;
        I.speculative = 0;
        pl.spec = false;
    }
    // The NEXT-3 jump kernel when forced, or by default (AUTO store) for too few streams to
    // fill the GPU; an explicit store path is honoured.
    const bool store_auto = (p->flags & PRNGD_STORE_MASK) == PRNGD_FLAG_STORE_AUTO;
    pl.jump = !mrg && ((p->flags & PRNGD_FLAG_JUMP) ||
                       (!(p->flags & PRNGD_FLAG_NO_JUMP) && !alg1 && store_auto &&
                        p->n_streams < 16384 && p->n_per_stream >= 512));
    switch (p->flags & PRNGD_STORE_MASK) {
        case PRNGD_FLAG_STORE_TMA: pl.store = Store::TMA; break;
        case PRNGD_FLAG_STORE_TILE: pl.store = Store::STG16; break;
        case PRNGD_FLAG_STORE_DIRECT: pl.store = Store::DIRECT; break;
        case PRNGD_FLAG_STORE_ROW1K: pl.store = Store::ROW1K; break;
        case PRNGD_FLAG_STORE_ROW: pl.store = Store::ROW; break;
        case PRNGD_FLAG_STORE_SEG: pl.store = Store::SEG; break;
        case PRNGD_FLAG_STORE_SEGC: pl.store = Store::SEGC; break;
        default: pl.store = Store::ROW; break;  // AUTO: ROW; plan_for may pick SEG (below)
    }
    pl.store_auto = store_auto;
    pl.exact_hist = (p->flags & PRNGD_FLAG_EXACT_HIST) != 0;
    *out = h;
    return PRNGD_OK;
}

prngd_status prngd_destroy(prngd_handle *h) {
    if (!h) return PRNGD_OK;
    if (h->scratch_dev >= 0) {
        int cur = -1;
        cudaGetDevice(&cur);
        cudaSetDevice(h->scratch_dev);
        if (h->cons_scratch) cudaFree(h->cons_scratch);
        for (int i = 0; i < 2; ++i) {
            if (h->stage[i]) cudaFree(h->stage[i]);
            if (h->ev_gen[i]) cudaEventDestroy(h->ev_gen[i]);
            if (h->ev_copy[i]) cudaEventDestroy(h->ev_copy[i]);
        }
        if (h->ev_stage_free) cudaEventDestroy(h->ev_stage_free);
        if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
        if (cur >= 0) cudaSetDevice(cur);
    }
    delete h;
    return PRNGD_OK;
}

static Plan plan_for(const prngd_handle *h, const void *out, bool consume = false);

prngd_status prngd_get_info(const prngd_handle *h, prngd_info *info) {
    if (!h || !info) return fail(PRNGD_EINVAL, "null argument");
    *info = h->info;
    const Plan pl = plan_for(h, reinterpret_cast<const void *>(uintptr_t{256}));
    info->store = (uint32_t)pl.store;
    info->kernel = pl.mrg ? 3u
                   : pl.jump ? (prngd::jump_uses_narrow_kernel(h->args) ? 5u : 2u)
                   : pl.store == Store::SEG ? 1u
                   : pl.store == Store::SEGC ? 4u : 0u;
    return PRNGD_OK;
}

uint32_t prngd_last_launches(const prngd_handle *h) { return h ? h->last_launches.load() : 0u; }

// Store path for this output pointer: the requested one when its alignment rules hold, else
// the next one that is legal (same bits whichever path writes them).
static Plan plan_for(const prngd_handle *h, const void *out, bool consume) {
    Plan pl = h->plan;
    // Fused consumer + outputs: the ROW tiles of consume_kernel next to its 128 KiB histogram
    // (S7).
    const uintptr_t a = (uintptr_t)out;
    const uint64_t nps = h->p.n_per_stream;
    const bool a32 = (a & 31u) == 0 && (nps & 3u) == 0;
    const bool a16 = (a & 15u) == 0 && (nps & 1u) == 0;
#ifndef PRNGD_CONS_SEG
#define PRNGD_CONS_SEG 1  // fused consumer with 1 KiB row segments where they apply
#endif
    if (consume && (pl.store == Store::SEG || pl.store == Store::SEGC || pl.store_auto)) {
        // the row-segment consumer needs rare rejection, pair-drop, 16-byte stores and
        // nps = 128 * 2^m <= 4096 (the kernel also checks the mapping); else ROW tiles
        const uint64_t S = nps / 128u;
        const bool seg = PRNGD_CONS_SEG && !pl.mrg && pl.spec && !pl.alg1 && !pl.ieee_div && a16 &&
                         nps % 128u == 0 && S >= 1 && S <= 32 && (S & (S - 1)) == 0;
        pl.store = seg ? Store::SEG : Store::ROW;
        pl.jump = false;
    }
    if (consume) {  // an explicit store path for the consumer, with the same alignment fallbacks
        if (pl.store == Store::SEG) return pl;  // checked above
        if ((pl.store == Store::ROW || pl.store == Store::ROW1K) && !a16) pl.store = Store::STG8;
#if PRNGD_AB_STORES
        if (pl.store == Store::DIRECT && !a32) pl.store = a16 ? Store::STG16 : Store::STG8;
        if (pl.store == Store::STG16 && !a16) pl.store = Store::STG8;
        if (pl.store == Store::TMA && !a16) pl.store = Store::STG8;
#endif
        return pl;
    }
    // SEG: rare rejection (speculative), pair-drop, nps = 128 * S with S a power of two <= 32,
    // and 16-byte stores; otherwise the ROW path.  AUTO takes SEG instead of the NEXT-3 jump
    // kernel for few-stream generate calls (cfg1: 76 vs 64 Gd/s); for bulk shapes ROW stays
    // ahead (cfg3: 790 vs 645 Gd/s: the per-segment jump costs more than the store pattern
    // gains).
    // segment length: 128 outputs (1 KiB, the measured best store pattern) unless the grid
    // would not fill one wave of resident warps (148 SMs x 12), then the shortest of 64 / 32
    // that the row length allows (more lanes per row, a shorter serial chain per lane)
    auto seg_fits = [&](uint64_t so) {
        const uint64_t S = nps / so;
        return nps % so == 0 && S >= 1 && S <= 32 && (S & (S - 1)) == 0;
    };
    pl.seg_out = 0;
    for (uint64_t so : {128ull, 64ull, 32ull}) {
        if (!seg_fits(so)) continue;
        pl.seg_out = (uint32_t)so;
        const uint64_t warps = h->p.n_streams * (nps / so) / 32u;
        if (warps >= 148ull * 12) break;
    }
    const bool seg_ok = !pl.mrg && pl.spec && !pl.alg1 && a16 && pl.seg_out != 0;
    if (pl.store == Store::SEG && !seg_ok) pl.store = Store::ROW;
    // SEGC: the same conditions with 8 column blocks of a multiple of 64 outputs each
    const bool segc_ok = !pl.mrg && pl.spec && !pl.alg1 && a16 && nps % 512 == 0;
    if (pl.store == Store::SEGC && !segc_ok) pl.store = Store::ROW;
    if (!consume && pl.store_auto && pl.jump && !(h->p.flags & PRNGD_FLAG_JUMP) && seg_ok) {
        pl.jump = false;
        pl.store = Store::SEG;
    }
    if ((pl.store == Store::ROW || pl.store == Store::ROW1K) && !a16) pl.store = Store::STG8;
#if PRNGD_AB_STORES
    const bool tma_ok = a16 && h->p.n_streams < (1ull << 31) && nps < (1ull << 31);
    if (pl.store == Store::DIRECT && !a32) pl.store = a16 ? Store::STG16 : Store::STG8;
    if (pl.store == Store::TMA && !tma_ok) pl.store = a16 ? Store::STG16 : Store::STG8;
    if (pl.store == Store::STG16 && !a16) pl.store = Store::STG8;
#else
    (void)a32;
#endif
    return pl;
}

// xorshift128 generate kernels: NEXT-3 jump (a warp per stream), SEG (a lane per row segment),
// or one lane per stream (ROW / STG8).
static cudaError_t launch_rows(const GenArgs &g, const Plan &pl, cudaStream_t st, int sms) {
    if (pl.jump) return prngd::launch_generate_jump(g, pl, st);
    if (pl.store == Store::SEGC) return prngd::launch_generate_segc(g, pl, st);
    if (pl.store == Store::SEG) return prngd::launch_generate_seg(g, pl, st);
    return prngd::launch_generate(g, pl, st, sms);
}

prngd_status prngd_generate(const prngd_handle *h, double *d_out, void *cuda_stream) {
    NvtxRange nvtx_range("prngd_generate");
    if (!h || !d_out) return fail(PRNGD_EINVAL, "null handle or output pointer");
    if ((uintptr_t)d_out & 7u) return fail(PRNGD_EINVAL, "d_out must be 8-byte aligned");
    int sms = 0;
    prngd_status s = device_ready(&sms);
    if (s != PRNGD_OK) return s;
    GenArgs g = h->args;
    g.out = d_out;
    cudaError_t e;
    const Plan pl = plan_for(h, d_out);
    if (pl.mrg) {
        if (pl.store != Store::ROW && pl.store != Store::ROW1K)
            return fail(PRNGD_EUNSUPPORTED, "MRG32k3a needs a 16-byte aligned output and even n_per_stream");
        e = prngd::launch_generate_mrg(g, pl.alg1, (cudaStream_t)cuda_stream);
    } else {
        e = launch_rows(g, pl, (cudaStream_t)cuda_stream, sms);
    }
    if (e != cudaSuccess) return cuda_fail(e, "generate kernel launch");
    h->last_launches.store(1);
    return PRNGD_OK;
}

static prngd_status ensure_device_scratch(prngd_handle *h) {
    int dev = -1;
    cudaGetDevice(&dev);
    if (h->scratch_dev >= 0 && h->scratch_dev != dev)
        return fail(PRNGD_EINVAL, "handle scratch lives on device %d, current device is %d",
                    h->scratch_dev, dev);
    h->scratch_dev = dev;
    return PRNGD_OK;
}

// Device staging buffers of whole warp tasks: generate_host keeps two of about 256 MiB in
// flight; the MRG32k3a consume-only path uses one of about 1 GiB (a 256 MiB chunk of a 1024-output
// shape is only 1024 one-warp CTAs, 40% of one wave).  *rows = streams per buffer.
static prngd_status ensure_stage(prngd_handle *h, uint64_t target, int nbuf, uint64_t *rows_out) {
    const uint64_t row_bytes = h->p.n_per_stream * 8u;
    uint64_t rows = target / row_bytes;
    if (rows < 1) rows = 1;
    if (rows >= 32) rows = rows / 32 * 32;  // whole warp tasks when the target holds them
    // (the kernels handle a partial last warp, so long rows just take fewer, not 32, per chunk)
    if (rows > h->p.n_streams) rows = h->p.n_streams;
    for (int i = 0; i < nbuf; ++i) {
        if (h->stage_rows[i] >= rows) continue;
        if (h->stage[i]) cudaFree(h->stage[i]);
        h->stage[i] = nullptr;
        h->stage_rows[i] = 0;
        const cudaError_t e = cudaMalloc(&h->stage[i], rows * row_bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(PRNGD_ENOMEM, "staging buffer (%llu bytes): %s",
                        (unsigned long long)(rows * row_bytes), cudaGetErrorString(e));
        }
        h->stage_rows[i] = rows;
    }
    *rows_out = rows;
    return PRNGD_OK;
}

// The staging buffers may still be read by an earlier MRG32k3a consume-only call on another
// stream: order this stream after it.
static prngd_status wait_stage_free(prngd_handle *h, cudaStream_t st) {
    if (!h->stage_pending) return PRNGD_OK;
    cudaError_t e = cudaStreamWaitEvent(st, h->ev_stage_free, 0);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent (staging buffer)");
    return PRNGD_OK;
}

static prngd_status generate_consume_impl(const prngd_handle *hc, double *d_out, int64_t *d_hist,
                                          double *d_pow, int64_t *d_count, uint64_t *d_arrive,
                                          bool mc, void *cuda_stream);

prngd_status prngd_generate_consume(const prngd_handle *hc, double *d_out, int64_t *d_hist,
                                    double *d_pow, int64_t *d_count, void *cuda_stream) {
    return generate_consume_impl(hc, d_out, d_hist, d_pow, d_count, nullptr, false, cuda_stream);
}

prngd_status prngd_generate_consume_ex(const prngd_handle *hc, double *d_out, int64_t *d_hist,
                                       double *d_pow, int64_t *d_count, uint64_t *d_arrive,
                                       void *cuda_stream) {
    return generate_consume_impl(hc, d_out, d_hist, d_pow, d_count, d_arrive, false, cuda_stream);
}

prngd_status prngd_generate_consume_mc(const prngd_handle *hc, double *d_out, void *mc_stats,
                                       void *cuda_stream) {
    if (!mc_stats || ((uintptr_t)mc_stats & 7u))
        return fail(PRNGD_EINVAL, "null or misaligned multicast statistics address");
    uint8_t *b = static_cast<uint8_t *>(mc_stats);
    return generate_consume_impl(hc, d_out, reinterpret_cast<int64_t *>(b),
                                 reinterpret_cast<double *>(b + PRNGD_STATS_POW_OFFSET),
                                 reinterpret_cast<int64_t *>(b + PRNGD_STATS_COUNT_OFFSET),
                                 reinterpret_cast<uint64_t *>(b + PRNGD_STATS_ARRIVE_OFFSET), true,
                                 cuda_stream);
}

static prngd_status generate_consume_impl(const prngd_handle *hc, double *d_out, int64_t *d_hist,
                                          double *d_pow, int64_t *d_count, uint64_t *d_arrive,
                                          bool mc, void *cuda_stream) {
    NvtxRange nvtx_range("prngd_generate_consume");
    if (!hc || !d_hist || !d_count)  // d_pow == NULL: histogram-only call
        return fail(PRNGD_EINVAL, "null handle or accumulator pointer");
    if (((uintptr_t)d_hist | (uintptr_t)d_pow | (uintptr_t)d_count | (uintptr_t)d_arrive) & 7u)
        return fail(PRNGD_EINVAL, "accumulators must be 8-byte aligned");
    unsigned long long *arrive = reinterpret_cast<unsigned long long *>(d_arrive);
    if (d_out && ((uintptr_t)d_out & 7u)) return fail(PRNGD_EINVAL, "d_out must be 8-byte aligned");
    int sms = 0;
    prngd_status s = device_ready(&sms);
    if (s != PRNGD_OK) return s;
    prngd_handle *h = const_cast<prngd_handle *>(hc);  // scratch is internal, behind the mutex
    std::lock_guard<std::mutex> lock(h->mu);
    if ((s = ensure_device_scratch(h)) != PRNGD_OK) return s;
    const size_t need = prngd::consume_scratch_bytes(sms);
    if (h->cons_bytes < need) {
        if (h->cons_scratch) cudaFree(h->cons_scratch);
        h->cons_scratch = nullptr;
        h->cons_bytes = 0;
        cudaError_t e = cudaMalloc(&h->cons_scratch, need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(PRNGD_ENOMEM, "consume scratch (%zu bytes): %s", need, cudaGetErrorString(e));
        }
        e = cudaMemset(h->cons_scratch, 0, need);  // the spill array must start at zero
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemset scratch");
        h->cons_bytes = need;
    }
    int launches = 0;
#ifndef PRNGD_MRG_FUSED
#define PRNGD_MRG_FUSED 1  // 0: generate, then read the values back (round-1 path, A/B only)
#endif
    if (mc && h->plan.mrg && !PRNGD_MRG_FUSED)
        return fail(PRNGD_EUNSUPPORTED, "multicast statistics need the fused MRG32k3a consumer");
    if (h->plan.mrg && PRNGD_MRG_FUSED) {
        // S7 fused into the MRG32k3a generator (consume_mrg_kernel): no read-back, no staging
        cudaError_t e = prngd::launch_generate_consume_mrg(
            h->args, h->plan.alg1, d_out, d_hist, d_pow, d_count, arrive, mc, h->cons_scratch,
            h->cons_bytes, (cudaStream_t)cuda_stream, sms, &launches);
        if (e != cudaSuccess) return cuda_fail(e, "generate_consume (MRG32k3a) launch");
        h->last_launches.store((uint32_t)launches);
        return PRNGD_OK;
    }
    if (h->plan.mrg) {
        // MRG32k3a: the generator kernel writes the values (d_out, or staged chunks when d_out
        // is null), then S7 runs over them in memory (launch_consume_memory)
        cudaStream_t st = (cudaStream_t)cuda_stream;
        const uint64_t nps = h->p.n_per_stream;
        uint64_t rows = h->p.n_streams;
        if (!d_out) {
            if ((s = ensure_stage(h, 1ull << 30, 1, &rows)) != PRNGD_OK) return s;
            if ((s = wait_stage_free(h, st)) != PRNGD_OK) return s;
        }
        for (uint64_t r0 = 0; r0 < h->p.n_streams; r0 += rows) {
            const uint64_t nr = (h->p.n_streams - r0) < rows ? (h->p.n_streams - r0) : rows;
            GenArgs g = h->args;
            g.stream_begin = h->p.stream_begin + r0;
            g.n_streams = nr;
            g.out = d_out ? d_out : h->stage[0];
            const Plan pl = plan_for(h, g.out);
            if (pl.store != Store::ROW && pl.store != Store::ROW1K)
                return fail(PRNGD_EUNSUPPORTED,
                            "MRG32k3a needs a 16-byte aligned output and even n_per_stream");
            cudaError_t e = prngd::launch_generate_mrg(g, pl.alg1, st);
            if (e != cudaSuccess) return cuda_fail(e, "generate kernel launch");
            int l = 0;
            const bool last = r0 + nr >= h->p.n_streams;  // only the last chunk signals arrival
            e = prngd::launch_consume_memory(h->args, g.out, nr * nps, d_hist, d_pow, d_count,
                                             last ? arrive : nullptr, h->cons_scratch,
                                             h->cons_bytes, st, sms, &l);
            if (e != cudaSuccess) return cuda_fail(e, "consume launch");
            launches += 1 + l;
        }
        if (!d_out) {
            if (!h->ev_stage_free) {
                cudaError_t e = cudaEventCreateWithFlags(&h->ev_stage_free, cudaEventDisableTiming);
                if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
            }
            cudaError_t e = cudaEventRecord(h->ev_stage_free, st);
            if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
            h->stage_pending = true;
        }
        h->last_launches.store((uint32_t)launches);
        return PRNGD_OK;
    }
    cudaError_t e = prngd::launch_generate_consume(h->args, plan_for(h, d_out, true), d_out, d_hist,
                                                   d_pow, d_count, arrive, mc, h->cons_scratch,
                                                   h->cons_bytes, (cudaStream_t)cuda_stream, sms,
                                                   &launches);
    if (e != cudaSuccess) return cuda_fail(e, "generate_consume launch");
    h->last_launches.store((uint32_t)launches);
    return PRNGD_OK;
}

prngd_status prngd_generate_host(prngd_handle *h, double *h_out, void *cuda_stream) {
    NvtxRange nvtx_range("prngd_generate_host");
    if (!h || !h_out) return fail(PRNGD_EINVAL, "null handle or host pointer");
    int sms = 0;
    prngd_status s = device_ready(&sms);
    if (s != PRNGD_OK) return s;
    std::lock_guard<std::mutex> lock(h->mu);
    if ((s = ensure_device_scratch(h)) != PRNGD_OK) return s;
    const uint64_t nps = h->p.n_per_stream;
    const uint64_t row_bytes = nps * 8u;
    uint64_t rows = 0;
    if ((s = ensure_stage(h, 256ull << 20, 2, &rows)) != PRNGD_OK) return s;
    cudaError_t e;
    if (!h->copy_stream) {
        if ((e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamCreate");
        for (int i = 0; i < 2; ++i) {
            if ((e = cudaEventCreateWithFlags(&h->ev_gen[i], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&h->ev_copy[i], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "cudaEventCreate");
        }
    }
    cudaStream_t gs = (cudaStream_t)cuda_stream;
    if ((s = wait_stage_free(h, gs)) != PRNGD_OK) return s;
    uint32_t launches = 0;
    bool used[2] = {false, false};
    for (uint64_t r0 = 0, c = 0; r0 < h->p.n_streams; r0 += rows, ++c) {
        const int b = (int)(c & 1u);
        const uint64_t nr = (h->p.n_streams - r0) < rows ? (h->p.n_streams - r0) : rows;
        if (used[b] && (e = cudaStreamWaitEvent(gs, h->ev_copy[b], 0)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamWaitEvent");
        GenArgs g = h->args;
        g.stream_begin = h->p.stream_begin + r0;
        g.n_streams = nr;
        g.out = h->stage[b];
        const Plan pl = plan_for(h, h->stage[b]);
        if (pl.mrg && pl.store != Store::ROW && pl.store != Store::ROW1K)
            return fail(PRNGD_EUNSUPPORTED, "MRG32k3a needs an even n_per_stream");
        e = pl.mrg ? prngd::launch_generate_mrg(g, pl.alg1, gs) : launch_rows(g, pl, gs, sms);
        // (launch_rows honours pl.jump, so prngd_get_info's kernel is the one that runs)
        if (e != cudaSuccess) return cuda_fail(e, "generate kernel launch");
        ++launches;
        if ((e = cudaEventRecord(h->ev_gen[b], gs)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
        if ((e = cudaStreamWaitEvent(h->copy_stream, h->ev_gen[b], 0)) != cudaSuccess)
            return cuda_fail(e, "cudaStreamWaitEvent");
        if ((e = cudaMemcpyAsync(h_out + r0 * nps, h->stage[b], nr * row_bytes,
                                 cudaMemcpyDeviceToHost, h->copy_stream)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpyAsync D2H");
        if ((e = cudaEventRecord(h->ev_copy[b], h->copy_stream)) != cudaSuccess)
            return cuda_fail(e, "cudaEventRecord");
        used[b] = true;
    }
    if ((e = cudaStreamSynchronize(h->copy_stream)) != cudaSuccess)
        return cuda_fail(e, "device->host pipeline");
    h->last_launches.store(launches);
    return PRNGD_OK;
}

prngd_status prngd_debug_raw(const prngd_handle *h, uint32_t *d_raw, uint64_t draws,
                             void *cuda_stream) {
    if (!h || !d_raw || draws == 0) return fail(PRNGD_EINVAL, "null argument or zero draws");
    if (h->plan.mrg) return fail(PRNGD_EUNSUPPORTED, "debug_raw dumps xorshift128 draws only");
    int sms = 0;
    prngd_status s = device_ready(&sms);
    if (s != PRNGD_OK) return s;
    cudaError_t e = prngd::launch_debug_raw(h->args, d_raw, draws, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "debug_raw launch");
    h->last_launches.store(1);
    return PRNGD_OK;
}

prngd_status prngd_debug_pairs(const prngd_handle *h, uint32_t *d_pair_index,
                               uint64_t *d_pairs_consumed, void *cuda_stream) {
    if (!h) return fail(PRNGD_EINVAL, "null handle");
    if (h->plan.mrg) return fail(PRNGD_EUNSUPPORTED, "debug_pairs follows xorshift128 only");
    int sms = 0;
    prngd_status s = device_ready(&sms);
    if (s != PRNGD_OK) return s;
    cudaError_t e = prngd::launch_debug_pairs(h->args, h->plan, d_pair_index, d_pairs_consumed,
                                              (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "debug_pairs launch");
    h->last_launches.store(1);
    return PRNGD_OK;
}

prngd_status prngd_debug_map(const prngd_handle *h, const uint32_t *d_x1, const uint32_t *d_x2,
                             double *d_z, uint64_t n, void *cuda_stream) {
    if (!h) return fail(PRNGD_EINVAL, "null handle");
    if (n && (!d_x1 || !d_x2 || !d_z)) return fail(PRNGD_EINVAL, "null array");
    int sms = 0;
    prngd_status s = device_ready(&sms);
    if (s != PRNGD_OK) return s;
    cudaError_t e = prngd::launch_debug_map(h->args, h->plan, d_x1, d_x2, d_z, n,
                                            (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "debug_map launch");
    h->last_launches.store(n ? 1 : 0);
    return PRNGD_OK;
}

prngd_status prngd_debug_jump(uint64_t n_draws, const uint32_t *in, uint32_t *out,
                              int lane_table) {
    if (!in || !out || lane_table > 31) return fail(PRNGD_EINVAL, "null state or lane > 31");
    prngd::jump_host(n_draws, in, out, lane_table);
    return PRNGD_OK;
}

prngd_status prngd_debug_div_check(const prngd_handle *h, uint64_t n, uint64_t seed,
                                   unsigned long long *d_mismatch, void *cuda_stream) {
    if (!h || !d_mismatch) return fail(PRNGD_EINVAL, "null argument");
    int sms = 0;
    prngd_status s = device_ready(&sms);
    if (s != PRNGD_OK) return s;
    cudaError_t e = prngd::launch_debug_div_check(h->args, n, seed, d_mismatch,
                                                  (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "debug_div_check launch");
    h->last_launches.store(n ? 1 : 0);
    return PRNGD_OK;
}

prngd_status prngd_wait_arrivals(const uint64_t *d_arrive, uint64_t target, uint64_t timeout_ns,
                                 void *cuda_stream) {
    NvtxRange nvtx_range("prngd_wait_arrivals");
    if (!d_arrive || ((uintptr_t)d_arrive & 7u)) return fail(PRNGD_EINVAL, "null or misaligned counter");
    cudaError_t e = prngd::launch_wait_arrivals(
        reinterpret_cast<const unsigned long long *>(d_arrive), target,
        timeout_ns ? timeout_ns : 60ull * 1000000000ull, (cudaStream_t)cuda_stream);
    return e == cudaSuccess ? PRNGD_OK : cuda_fail(e, "wait_arrivals launch");
}

prngd_status prngd_peer_alloc(uint64_t bytes, void **d_ptr) {
    if (!d_ptr || bytes == 0) return fail(PRNGD_EINVAL, "null pointer or zero size");
    *d_ptr = nullptr;
    cudaError_t e = cudaMalloc(d_ptr, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(PRNGD_ENOMEM, "peer accumulator (%llu bytes): %s", (unsigned long long)bytes,
                    cudaGetErrorString(e));
    }
    if ((e = cudaMemset(*d_ptr, 0, bytes)) != cudaSuccess) return cuda_fail(e, "cudaMemset");
    return PRNGD_OK;
}

prngd_status prngd_peer_free(void *d_ptr) {
    if (!d_ptr) return PRNGD_OK;
    cudaError_t e = cudaFree(d_ptr);
    return e == cudaSuccess ? PRNGD_OK : cuda_fail(e, "cudaFree");
}

prngd_status prngd_ipc_export(void *d_ptr, void *handle_out) {
    static_assert(sizeof(cudaIpcMemHandle_t) == PRNGD_IPC_HANDLE_BYTES, "IPC handle size");
    if (!d_ptr || !handle_out) return fail(PRNGD_EINVAL, "null argument");
    cudaIpcMemHandle_t hnd;
    cudaError_t e = cudaIpcGetMemHandle(&hnd, d_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    std::memcpy(handle_out, &hnd, sizeof(hnd));
    return PRNGD_OK;
}

prngd_status prngd_ipc_open(const void *handle, void **d_ptr) {
    if (!handle || !d_ptr) return fail(PRNGD_EINVAL, "null argument");
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, handle, sizeof(hnd));
    *d_ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(d_ptr, hnd, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? PRNGD_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

prngd_status prngd_ipc_close(void *d_ptr) {
    if (!d_ptr) return PRNGD_OK;
    cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
    return e == cudaSuccess ? PRNGD_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

prngd_status prngd_copy(void *dst, const void *src, uint64_t bytes, void *cuda_stream) {
    if ((!dst || !src) && bytes) return fail(PRNGD_EINVAL, "null pointer");
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)cuda_stream);
    return e == cudaSuccess ? PRNGD_OK : cuda_fail(e, "cudaMemcpyAsync");
}

prngd_status prngd_zero(void *d_ptr, uint64_t bytes, void *cuda_stream) {
    if (!d_ptr && bytes) return fail(PRNGD_EINVAL, "null pointer");
    cudaError_t e = cudaMemsetAsync(d_ptr, 0, bytes, (cudaStream_t)cuda_stream);
    return e == cudaSuccess ? PRNGD_OK : cuda_fail(e, "cudaMemsetAsync");
}

}  // extern "C"
