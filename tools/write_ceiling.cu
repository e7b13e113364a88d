// write_ceiling.cu -- B13 store-roofline microbenchmarks (measurement tool, not the product).
// All modes write incompressible 64-bit values (a cheap per-element hash, so L2 compression
// cannot shrink the DRAM traffic) into an n-double buffer:
//   mode 0  contiguous, grid-stride, 16-byte st.global.v2 (148 x 8 CTAs of 256)
//   mode 1  contiguous, grid-stride, 32-byte st.global.v4
//   mode 2  the generator's access pattern without its arithmetic: buffer viewed as
//           [rows][cols], one warp per 32 rows, 128 bytes of each row per step, warp-coalesced
//           16-byte stores (4 rows x 128 B per instruction), 4 warps per CTA, one CTA per 128 rows
//   mode 3  contiguous 16 KiB cp.async.bulk (TMA bulk) stores from shared memory
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double hval(uint64_t i, uint64_t salt) {
    uint32_t lo = (uint32_t)(i + salt) * 0x9E3779B1u;
    uint32_t hi = (lo ^ (lo >> 15)) * 0x85EBCA77u;
    return __hiloint2double((int)(hi & 0x3FEFFFFFu), (int)lo);
}

template <int VEC>
__global__ void __launch_bounds__(256) contiguous(double *p, uint64_t n, uint64_t salt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * VEC;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC; i + VEC <= n;
         i += stride) {
        if (VEC == 2)
            asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p + i), "d"(hval(i, salt)),
                         "d"(hval(i + 1, salt))
                         : "memory");
        else
            asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p + i),
                         "d"(hval(i, salt)), "d"(hval(i + 1, salt)), "d"(hval(i + 2, salt)),
                         "d"(hval(i + 3, salt))
                         : "memory");
    }
}

__global__ void __launch_bounds__(128) row_tiles(double *p, uint64_t rows, uint64_t cols,
                                                 uint64_t salt) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t row0 = ((uint64_t)blockIdx.x * 4 + warp) * 32;
    if (row0 >= rows) return;
    for (uint64_t c0 = 0; c0 + 16 <= cols; c0 += 16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint64_t r = row0 + k * 4 + (lane >> 3), c = c0 + 2 * (lane & 7u);
            double *q = p + r * cols + c;
            asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(q), "d"(hval(r * cols + c, salt)),
                         "d"(hval(r * cols + c + 1, salt))
                         : "memory");
        }
    }
}

__global__ void __launch_bounds__(128) bulk_contiguous(double *p, uint64_t n, uint64_t salt) {
    constexpr int kChunk = 16384;  // bytes per bulk store
    __shared__ alignas(128) double buf[2][kChunk / 8];
    for (int i = threadIdx.x; i < 2 * kChunk / 8; i += blockDim.x)
        (&buf[0][0])[i] = hval(blockIdx.x * 4096u + i, salt);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint64_t chunks = n * 8 / kChunk;
    int k = 0;
    for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x, k ^= 1) {
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[k][0]);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         p + c * (kChunk / 8)),
                     "r"(s), "n"(kChunk)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// The generator's row-major [rows][1024] layout, one warp per 32 rows, but each row receives
// `burst` contiguous bytes at a time (the warp writes one row's burst back to back, 512 B per
// instruction), so DRAM sees bursts of that size per row.  Occupancy can be limited with
// dynamic shared memory padding.
__global__ void __launch_bounds__(128) row_bursts(double *p, uint64_t rows, uint64_t cols,
                                                  uint32_t burst_doubles, uint64_t salt) {
    extern __shared__ uint8_t pad[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t row0 = ((uint64_t)blockIdx.x * 4 + warp) * 32;
    if (row0 >= rows) return;
    if (salt == ~0ull) pad[threadIdx.x] = 0;  // keep the smem allocation alive
    for (uint64_t c0 = 0; c0 < cols; c0 += burst_doubles) {
        for (uint32_t r = 0; r < 32; ++r) {
            for (uint32_t k = 2 * lane; k < burst_doubles; k += 64) {
                const uint64_t e = (row0 + r) * cols + c0 + k;
                asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p + e), "d"(hval(e, salt)),
                             "d"(hval(e + 1, salt))
                             : "memory");
            }
        }
    }
}

extern "C" __attribute__((visibility("default"))) int wc_pattern(double *p, uint64_t n,
                                                                 uint32_t burst_bytes,
                                                                 uint32_t smem_pad, uint64_t salt,
                                                                 void *stream) {
    const uint64_t cols = 1024, rows = n / cols;
    cudaFuncSetAttribute(row_bursts, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    row_bursts<<<(unsigned)((rows + 127) / 128), 128, smem_pad, (cudaStream_t)stream>>>(
        p, rows, cols, burst_bytes / 8, salt);
    return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) int wc_store(double *p, uint64_t n, int mode,
                                                               uint64_t salt, void *stream) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t st = (cudaStream_t)stream;
    switch (mode) {
        case 0: contiguous<2><<<sms * 8, 256, 0, st>>>(p, n, salt); break;
        case 1: contiguous<4><<<sms * 8, 256, 0, st>>>(p, n, salt); break;
        case 2: {  // rows x 1024 columns, like cfg3
            const uint64_t cols = 1024, rows = n / cols;
            row_tiles<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(p, rows, cols, salt);
            break;
        }
        case 3: bulk_contiguous<<<sms * 4, 128, 0, st>>>(p, n, salt); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}

// Segmented rows: the buffer is [rows][cols]; a one-warp CTA owns 32/S rows, each split into S
// segments (lane = row_local * S + seg owns one segment).  Each flush writes `chunk` bytes of
// every segment (32 chunks per flush, 512 B per instruction walking the chunks in lane order),
// so S = 1, chunk = 512 is the ROW kernel's pattern and S = 32, chunk = cols*8/32 writes one
// whole row per flush.  Occupancy is set by the dynamic smem pad (the real tile size).
__global__ void __launch_bounds__(32) row_segments(double *p, uint64_t rows, uint64_t cols,
                                                   uint32_t S, uint32_t chunk_doubles,
                                                   uint64_t salt) {
    extern __shared__ uint8_t pad[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t rpw = 32u / S;
    const uint64_t row0 = (uint64_t)blockIdx.x * rpw;
    if (row0 >= rows) return;
    if (salt == ~0ull) pad[threadIdx.x] = 0;
    const uint64_t seg_len = cols / S;
    const uint32_t per_flush = 32u * chunk_doubles;  // doubles per flush
    for (uint64_t v = 0; v * chunk_doubles < seg_len; ++v) {
        for (uint32_t off = 2 * lane; off < per_flush; off += 64) {
            const uint32_t c = off / chunk_doubles, within = off % chunk_doubles;
            const uint64_t r = row0 + c / S, seg = c % S;
            const uint64_t e = r * cols + seg * seg_len + v * chunk_doubles + within;
            asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p + e), "d"(hval(e, salt)),
                         "d"(hval(e + 1, salt))
                         : "memory");
        }
    }
}

extern "C" __attribute__((visibility("default"))) int wc_segments(double *p, uint64_t n,
                                                                  uint32_t S, uint32_t chunk_bytes,
                                                                  uint32_t smem_pad, uint64_t salt,
                                                                  void *stream, uint64_t cols) {
    const uint64_t rows = n / cols;
    cudaFuncSetAttribute(row_segments, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const uint32_t rpw = 32u / S;
    row_segments<<<(unsigned)((rows + rpw - 1) / rpw), 32, smem_pad, (cudaStream_t)stream>>>(
        p, rows, cols, S, chunk_bytes / 8, salt);
    return (int)cudaGetLastError();
}

// Rotated rows: the ROW kernel's pattern (one lane per row, 512-byte chunks) but lane r runs
// its rows with a column phase: over M rows per lane (rows base + 32 m + r), at flush step t
// lane r writes chunk (t + d_r) mod C of its current row, d_r = (r * skew) mod C, so one flush
// touches many column offsets (address bits below the row size) instead of one.
template <uint32_t C, uint32_t M>
__global__ void __launch_bounds__(32) rot_rows(double *p, uint64_t rows, uint64_t cols,
                                               uint32_t skew, uint64_t salt) {
    extern __shared__ uint8_t pad[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t base = (uint64_t)blockIdx.x * 32u * M;
    if (base >= rows) return;
    if (salt == ~0ull) pad[threadIdx.x] = 0;
    for (uint32_t t = 0; t < M * C; ++t) {
#pragma unroll 4
        for (uint32_t r = 0; r < 32; ++r) {
            const uint32_t d = (r * skew) & (C - 1);
            const uint32_t v = (t + d) & (M * C - 1);  // position in lane r's row sequence
            const uint64_t row = base + 32u * (v / C) + r;
            const uint64_t e = row * cols + (uint64_t)(v & (C - 1)) * 64 + 2 * lane;
            if (row < rows)
                asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p + e), "d"(hval(e, salt)),
                             "d"(hval(e + 1, salt))
                             : "memory");
        }
    }
}

extern "C" __attribute__((visibility("default"))) int wc_rot(double *p, uint64_t n, uint32_t M,
                                                             uint32_t skew, uint32_t smem_pad,
                                                             uint64_t salt, void *stream,
                                                             uint64_t cols) {
    const uint64_t rows = n / cols;
    const uint64_t per = 32ull * M;
    const unsigned grid = (unsigned)((rows + per - 1) / per);
    cudaStream_t st = (cudaStream_t)stream;
#define ROT(CC, MM)                                                                             \
    if (cols / 64 == CC && M == MM) {                                                           \
        cudaFuncSetAttribute(rot_rows<CC, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             200 * 1024);                                                       \
        rot_rows<CC, MM><<<grid, 32, smem_pad, st>>>(p, rows, cols, skew, salt);                \
        return (int)cudaGetLastError();                                                         \
    }
    ROT(16, 1) ROT(16, 4) ROT(32, 1) ROT(32, 4) ROT(64, 1) ROT(64, 4)
#undef ROT
    return -1;
}

// Block columns: a CTA of S warps owns 32 rows; warp w writes column block w (cols / S doubles)
// of every row, 512 bytes per row per flush (one row per instruction, like the ROW kernel), so
// a warp's flush is strided by the row length but the CTA completes its 32-row block within
// cols / S / 64 flushes.
__global__ void blockcol_rows(double *p, uint64_t rows, uint64_t cols, uint32_t chunk,
                              uint64_t salt) {
    extern __shared__ uint8_t pad[];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5, S = blockDim.x >> 5;
    const uint64_t row0 = (uint64_t)blockIdx.x * 32u;
    if (row0 >= rows) return;
    if (salt == ~0ull) pad[threadIdx.x] = 0;
    const uint64_t seg = cols / S;
    const uint32_t lpr = chunk / 16;  // lanes per row per instruction
    for (uint64_t c0 = 0; c0 < seg; c0 += chunk / 8) {
        for (uint32_t r = 0; r < 32; r += 32 / lpr) {
            const uint64_t row = row0 + r + lane / lpr;
            const uint64_t e = row * cols + w * seg + c0 + 2 * (lane % lpr);
            if (row < rows)
                asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p + e), "d"(hval(e, salt)),
                             "d"(hval(e + 1, salt))
                             : "memory");
        }
    }
}

extern "C" __attribute__((visibility("default"))) int wc_blockcol(double *p, uint64_t n,
                                                                  uint32_t S, uint32_t smem_pad,
                                                                  uint64_t salt, void *stream,
                                                                  uint64_t cols, uint32_t chunk) {
    const uint64_t rows = n / cols;
    cudaFuncSetAttribute(blockcol_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    blockcol_rows<<<(unsigned)((rows + 31) / 32), 32 * S, smem_pad, (cudaStream_t)stream>>>(
        p, rows, cols, chunk, salt);
    return (int)cudaGetLastError();
}

// Shared-memory histogram increment ceiling: every thread issues `iters` adds of 1 << 16*(b&1)
// into a 32768-word (128 KiB) packed histogram at pseudo-random bins b (xorshift32 per thread),
// RED (no return) when red != 0, else atomicAdd with its return value consumed.  One CTA of
// `warps` warps per SM (the fused consumer's shape).  Returns via *ops the total adds.
__global__ void smem_hist_rate(uint32_t iters, int red, unsigned long long *sink) {
    extern __shared__ uint32_t h[];
    for (uint32_t i = threadIdx.x; i < 32768; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1), acc = 0;
    for (uint32_t k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            const uint32_t b = x >> 16;
            const uint32_t inc = __funnelshift_l(1u, 1u, b << 4);
            if (red)
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&h[b >> 1])), "r"(inc) : "memory");
            else
                acc += atomicAdd(&h[b >> 1], inc);
        }
    }
    if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

extern "C" __attribute__((visibility("default"))) int wc_smem_hist(uint32_t iters, int red,
                                                                   int warps, void *stream,
                                                                   void *sink) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(smem_hist_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    smem_hist_rate<<<sms, warps * 32, 131072, (cudaStream_t)stream>>>(
        iters, red, (unsigned long long *)sink);
    return (int)cudaGetLastError();
}

// Distributed-shared-memory histogram adds: a cluster of C CTAs (one per SM) splits the 65536
// packed bins, CTA c owning bins [c*65536/C, (c+1)*65536/C) in (65536/C)/2 words; every thread
// adds to random bins wherever they live (red.shared::cluster into the owner's shared memory).
// Measures whether a cluster-split histogram can free shared memory at the consumer's rate.
__global__ void dsmem_hist_rate(uint32_t iters, unsigned long long *sink) {
    extern __shared__ uint32_t h[];
    uint32_t csize, crank;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const uint32_t words = 32768u / csize;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) h[i] = 0;
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(h);
    for (uint32_t k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            const uint32_t b = x >> 16;
            const uint32_t inc = __funnelshift_l(1u, 1u, b << 4);
            const uint32_t w = b >> 1;
            const uint32_t owner = w / words, off = (w - owner * words) * 4u;
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + off), "r"(owner));
            asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(ra), "r"(inc) : "memory");
        }
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (x == 0xFFFFFFFFu) sink[0] = x;
}

extern "C" __attribute__((visibility("default"))) int wc_dsmem_hist(uint32_t iters, int csize,
                                                                    int warps, void *stream,
                                                                    void *sink) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 131072 / csize;
    cudaFuncSetAttribute(dsmem_hist_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dsmem_hist_rate, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sms / csize * csize));
    cfg.blockDim = dim3(warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, dsmem_hist_rate, iters, (unsigned long long *)sink);
    return (int)cudaGetLastError();
}

// Per-lane rows: a one-warp CTA owns 32 rows, lane r writes ITS OWN row r, `burst` bytes at a
// time with 32-byte st.global.v4 (burst / 32 consecutive stores), then moves to the next burst
// of the row.  burst = 128 is the DIRECT store path's pattern (one 16-output batch from
// registers); burst = 512 / 1024 is what a lane could write after staging 64 / 128 outputs of
// its row off-register (e.g. in tensor memory).  Occupancy is set by the dynamic smem pad.
__global__ void __launch_bounds__(32) lane_rows(double *p, uint64_t rows, uint64_t cols,
                                                uint32_t burst_doubles, uint64_t salt) {
    extern __shared__ uint8_t pad[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t row = (uint64_t)blockIdx.x * 32u + lane;
    if (row >= rows) return;
    if (salt == ~0ull) pad[threadIdx.x] = 0;
    double *q = p + row * cols;
    for (uint64_t c0 = 0; c0 < cols; c0 += burst_doubles) {
#pragma unroll 4
        for (uint32_t k = 0; k < burst_doubles; k += 4) {
            const uint64_t e = row * cols + c0 + k;
            asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(q + c0 + k),
                         "d"(hval(e, salt)), "d"(hval(e + 1, salt)), "d"(hval(e + 2, salt)),
                         "d"(hval(e + 3, salt))
                         : "memory");
        }
    }
}

extern "C" __attribute__((visibility("default"))) int wc_lane_rows(double *p, uint64_t n,
                                                                   uint32_t burst_bytes,
                                                                   uint32_t smem_pad, uint64_t salt,
                                                                   void *stream, uint64_t cols) {
    const uint64_t rows = n / cols;
    cudaFuncSetAttribute(lane_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    lane_rows<<<(unsigned)((rows + 31) / 32), 32, smem_pad, (cudaStream_t)stream>>>(
        p, rows, cols, burst_bytes / 8, salt);
    return (int)cudaGetLastError();
}
