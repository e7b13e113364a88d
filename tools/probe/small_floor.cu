// Floor probes for the small configs (cfg1: 8 MiB, cfg2: 32 MiB of output per step): an empty
// launch and plain 16-byte store kernels with the same grid shapes, timed by small_floor.py
// under bench.py's L2-flush protocol.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void empty_kernel() {}

// one warp per contiguous row of `row_d2` double2 (the SEG / jump kernels' output shape)
__global__ void row_store_kernel(double2 *out, uint32_t row_d2, uint64_t n_rows) {
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (w >= n_rows) return;
    double2 *r = out + w * row_d2;
    for (uint32_t i = lane; i < row_d2; i += 32) r[i] = make_double2((double)i, (double)w);
}

// grid-stride 16-byte stores over the whole buffer
__global__ void flat_store_kernel(double2 *out, uint64_t n_d2) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_d2;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = make_double2((double)i, 1.0);
}

extern "C" int probe_empty(unsigned grid, unsigned block, void *st) {
    empty_kernel<<<grid, block, 0, (cudaStream_t)st>>>();
    return (int)cudaGetLastError();
}
extern "C" int probe_rows(void *out, uint32_t row_d2, uint64_t n_rows, unsigned warps_per_cta,
                          void *st) {
    const uint64_t grid = (n_rows + warps_per_cta - 1) / warps_per_cta;
    row_store_kernel<<<(unsigned)grid, 32 * warps_per_cta, 0, (cudaStream_t)st>>>(
        (double2 *)out, row_d2, n_rows);
    return (int)cudaGetLastError();
}
extern "C" int probe_flat(void *out, uint64_t n_d2, unsigned grid, unsigned block, void *st) {
    flat_store_kernel<<<grid, block, 0, (cudaStream_t)st>>>((double2 *)out, n_d2);
    return (int)cudaGetLastError();
}
