// Probe: does a single-device NVLS multicast object work here, and do multimem.red.add.{u64,f64}
// land in the bound physical memory?  nvcc -gencode arch=compute_100a,code=sm_100a mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)

__global__ void red_kernel(unsigned long long *mc, double *mcd, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(mc + i), "l"((unsigned long long)(i + 1)) : "memory");
        asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(mcd + i), "d"(0.5 * i) : "memory");
    }
}

int main() {
    CK(cuInit(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
    int mcs = 0; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("multicast supported: %d\n", mcs);
    const int n = 65536;
    size_t bytes = (size_t)n * 16;
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    prop.size = bytes;
    CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    bytes = (bytes + gran - 1) / gran * gran;
    prop.size = bytes;
    printf("granularity %zu, size %zu\n", gran, bytes);
    CUmemGenericAllocationHandle mc;
    for (unsigned nd : {1u, 2u}) for (unsigned long long ht : {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC}) {
        CUmulticastObjectProp p2 = prop; p2.numDevices = nd; p2.handleTypes = ht;
        CUresult r = cuMulticastCreate(&mc, &p2);
        const char *es; cuGetErrorString(r, &es);
        printf("create numDevices=%u handleTypes=%llu -> %s\n", nd, ht, es);
        if (r == CUDA_SUCCESS) cuMemRelease(mc);
    }
    prop.handleTypes = 0;
    CK(cuMulticastCreate(&mc, &prop));
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
    size_t pgran = 0; CK(cuMemGetAllocationGranularity(&pgran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    printf("phys granularity %zu\n", pgran);
    CUmemGenericAllocationHandle phys; CK(cuMemCreate(&phys, bytes, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, phys, 0, bytes, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, bytes, gran, 0, 0));
    CK(cuMemMap(uc, bytes, 0, phys, 0));
    CK(cuMemAddressReserve(&mcp, bytes, gran, 0, 0));
    CK(cuMemMap(mcp, bytes, 0, mc, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = dev; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, bytes, &ad, 1));
    CK(cuMemSetAccess(mcp, bytes, &ad, 1));
    CK(cuMemsetD8(uc, 0, bytes));
    red_kernel<<<64, 256>>>((unsigned long long *)mcp, (double *)(mcp + n * 8), n);
    red_kernel<<<64, 256>>>((unsigned long long *)mcp, (double *)(mcp + n * 8), n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    unsigned long long h[4]; double hd[4];
    CK(cuMemcpyDtoH(h, uc + 8 * 100, 32));
    CK(cuMemcpyDtoH(hd, uc + n * 8 + 8 * 100, 32));
    printf("u64[100..103] = %llu %llu %llu %llu (expect 202 204 206 208)\n", h[0], h[1], h[2], h[3]);
    printf("f64[100..103] = %g %g %g %g (expect 100 101 102 103)\n", hd[0], hd[1], hd[2], hd[3]);
    int fd = -1;
    CUresult r = cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    printf("export fd: %d (res %d)\n", fd, (int)r);
    return 0;
}
