// Shared-memory wavefront probe for the fused consumer's tile (S7): how many
// wavefronts do the per-lane STS.128 row writes and the 8-lanes-per-row LDS.128 flush reads of a
// 32-row tile cost at a given padded row stride, alone on the SM and beside random-bin
// red.shared adds (the histogram)?  Run under ncu with the l1tex shared wavefront / bank-conflict
// counters; one launch per (stride, with_atomics) variant, kernel names carry the variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_pattern lds_pattern.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void sts_v2(uint32_t a, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void lds_v2(uint32_t a, double &x, double &y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}

// RS: tile row stride in bytes; ATOM: also 16 random-bin red.shared.add.u32 per lane per batch
// (one per output, like the histogram); ROWS32: the bulk ROW flush (32 lanes read one row's 512 B,
// rows of 64 outputs) instead of the consumer's 8 lanes per 128-byte row.
template <int RS, bool ATOM, bool ROWS32, int WARPS = 1>
__global__ void __launch_bounds__(32 * WARPS) probe(double *out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t hist = base, tile = base + (ATOM ? 131072u : 0u) + warp * 32u * RS;
    constexpr int COLS = ROWS32 ? 64 : 16;
    uint32_t x = 0x9E3779B9u * (blockIdx.x * 32 * WARPS + threadIdx.x + 1);
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        const uint32_t my = tile + lane * RS;
#pragma unroll
        for (int c = 0; c < COLS / 2; ++c) sts_v2(my + (c << 4), (double)it, (double)c);
        if (ATOM) {
#pragma unroll
            for (int i = 0; i < COLS; ++i) {
                x ^= x << 13; x ^= x >> 17; x ^= x << 5;
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(hist + (x & 0x1FFFCu)), "r"(1u) : "memory");
            }
        }
        __syncwarp();
        if (ROWS32) {
#pragma unroll
            for (uint32_t r = 0; r < 32u; ++r) {
                double a0, a1;
                lds_v2(tile + r * RS + (lane << 4), a0, a1);
                acc += a0 + a1;
            }
        } else {
            const uint32_t c = lane & 7u, rsub = lane >> 3;
#pragma unroll
            for (uint32_t r = rsub; r < 32u; r += 4u) {
                double a0, a1;
                lds_v2(tile + r * RS + (c << 4), a0, a1);
                acc += a0 + a1;
            }
        }
        __syncwarp();
    }
    if (acc == -1.0) out[0] = acc;
}

template <int RS, bool ATOM, bool ROWS32, int WARPS = 1>
static void run(const char *name, double *out, int ctas) {
    const size_t smem = (ATOM ? 131072 : 0) + WARPS * 32 * RS + 1024;
    cudaFuncSetAttribute(probe<RS, ATOM, ROWS32, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<RS, ATOM, ROWS32, WARPS><<<ctas, 32 * WARPS, smem>>>(out, 1024);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s: %s\n", name, cudaGetErrorString(e));
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    // launch order = the order of the ncu rows
    run<144, false, false>("rs144", out, 148 * 4);
    run<176, false, false>("rs176", out, 148 * 4);
    run<208, false, false>("rs208", out, 148 * 4);
    run<272, false, false>("rs272", out, 148 * 4);
    run<128, false, false>("rs128 (unpadded)", out, 148 * 4);
    run<528, false, true>("rows32 rs528 (bulk ROW flush)", out, 148 * 4);
    run<144, true, false>("rs144 + red.shared", out, 148);
    run<176, true, false>("rs176 + red.shared", out, 148);
    run<528, true, true>("rows32 rs528 + red.shared", out, 148);
    // 16 warps per CTA beside one shared histogram, as in consume_kernel
    run<144, true, false, 16>("rs144 + red.shared, 16 warps", out, 148);
    run<144, false, false, 16>("rs144, 16 warps, no adds", out, 148);
    run<176, true, false, 16>("rs176 + red.shared, 16 warps", out, 148);
    return 0;
}
