// Probe: sustained pure-store HBM bandwidth when only S of the SMs issue the stores (one
// 1024-thread CTA per SM, forced by a large dynamic shared-memory request).  Question: under the
// board's power cap, does leaving SMs idle buy store bandwidth?
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double hv(uint64_t i, uint64_t salt) {
    uint32_t lo = (uint32_t)(i * 0x9E3779B1u) ^ (uint32_t)salt;
    uint32_t hi = (lo ^ (lo >> 15)) * 0x85EBCA77u;
    return __hiloint2double((int)(hi & 0x3FEFFFFFu), (int)lo);
}

__global__ void __launch_bounds__(1024, 1) stores(double *p, uint64_t n, uint64_t salt) {
    extern __shared__ uint8_t pad[];
    if (n == 0) pad[threadIdx.x] = 0;  // keep the allocation
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i + 4 <= n; i += stride)
        asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p + i), "d"(hv(i, salt)),
                     "d"(hv(i + 1, salt)), "d"(hv(i + 2, salt)), "d"(hv(i + 3, salt))
                     : "memory");
}

extern "C" __attribute__((visibility("default"))) int sm_stores(double *p, uint64_t n, int sms,
                                                                uint64_t salt, void *stream) {
    const size_t smem = 150 * 1024;
    cudaFuncSetAttribute(stores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    stores<<<sms, 1024, smem, (cudaStream_t)stream>>>(p, n, salt);
    return (int)cudaGetLastError();
}
