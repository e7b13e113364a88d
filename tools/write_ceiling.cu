// write_ceiling.cu -- B13 store-roofline microbenchmark (measurement tool, not the product).
// Streams incompressible 64-bit values (a per-element hash, so L2 compression cannot shrink the
// DRAM traffic) over a buffer with 16- or 32-byte coalesced stores, grid = 148 x occupancy.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t h64(uint64_t v) {
    v ^= v >> 33; v *= 0xff51afd7ed558ccdull; v ^= v >> 33; return v;
}

template <int VEC>
__global__ void __launch_bounds__(256) store_kernel(double *p, uint64_t n, uint64_t salt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * VEC;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC; i + VEC <= n; i += stride) {
        double v[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[k] = __longlong_as_double((long long)(h64(i + k + salt) >> 12));
        if (VEC == 2)
            asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" :: "l"(p + i), "d"(v[0]), "d"(v[1]) : "memory");
        else
            asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" :: "l"(p + i), "d"(v[0]), "d"(v[1]),
                         "d"(v[VEC > 2 ? 2 : 0]), "d"(v[VEC > 3 ? 3 : 0]) : "memory");
    }
}

extern "C" __attribute__((visibility("default"))) int wc_store(double *p, uint64_t n, int vec,
                                                               uint64_t salt, void *stream) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 8;
    if (vec == 4) store_kernel<4><<<grid, 256, 0, (cudaStream_t)stream>>>(p, n, salt);
    else store_kernel<2><<<grid, 256, 0, (cudaStream_t)stream>>>(p, n, salt);
    return (int)cudaGetLastError();
}
