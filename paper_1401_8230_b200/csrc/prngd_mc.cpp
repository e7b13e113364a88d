// prngd_mc.cpp -- NEXT-4: NVLS multicast accumulator for the multi-GPU statistics reduction
// (DESIGN.md section 5 "Multi-GPU").
//
// One multicast object of the NVSwitch fabric spans the R ranks' GPUs; every rank binds one
// physical buffer of its own device to it and maps both the multicast address (writes through it
// are performed by the switch on every member's copy) and its own copy (unicast).  The finalize
// kernel of prngd_generate_consume_mc then adds its statistics with multimem.red through the
// multicast address, so the NVSwitch reduces them into every rank's copy -- an all-reduce done
// inside the library's own kernel, without a collective call.  Used only when the driver can
// create a multicast object for the group (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and a
// successful cuMulticastCreate for >= 2 devices); paper_1401_8230_b200.dist falls back to the
// peer-memory (PeerStats) and NCCL reductions otherwise.
//
// The driver API is reached through cudaGetDriverEntryPoint (the library links only cudart).
// The multicast handle is shared between processes as a POSIX file descriptor, fetched by the
// other ranks with pidfd_getfd (the owner allows it with PR_SET_PTRACER).  Product code;
// independent of oracle/.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/prctl.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>

#include "prngd_internal.h"

namespace {

thread_local char g_mc_err[256] = "";

prngd_status mc_fail(prngd_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_mc_err, sizeof(g_mc_err), fmt, ap);
    va_end(ap);
    prngd::set_last_error(g_mc_err);
    return s;
}

struct Drv {
    CUresult (*GetErrorString)(CUresult, const char **) = nullptr;
    CUresult (*DeviceGet)(CUdevice *, int) = nullptr;
    CUresult (*DeviceGetAttribute)(int *, CUdevice_attribute, CUdevice) = nullptr;
    CUresult (*MulticastCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *) = nullptr;
    CUresult (*MulticastGetGranularity)(size_t *, const CUmulticastObjectProp *,
                                        CUmulticastGranularity_flags) = nullptr;
    CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle,
                                 size_t, size_t, unsigned long long) = nullptr;
    CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*MemCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *,
                          unsigned long long) = nullptr;
    CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*MemGetAllocationGranularity)(size_t *, const CUmemAllocationProp *,
                                            CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*MemAddressReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr,
                                  unsigned long long) = nullptr;
    CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                       unsigned long long) = nullptr;
    CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
    CUresult (*MemExportToShareableHandle)(void *, CUmemGenericAllocationHandle,
                                           CUmemAllocationHandleType, unsigned long long) = nullptr;
    CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle *, void *,
                                             CUmemAllocationHandleType) = nullptr;
    bool ok = false;
};

template <class F>
bool entry(const char *name, F &f) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
        return false;
    f = reinterpret_cast<F>(p);
    return true;
}

const Drv &drv() {
    static std::once_flag once;
    static Drv d;
    std::call_once(once, [] {
        d.ok = entry("cuGetErrorString", d.GetErrorString) && entry("cuDeviceGet", d.DeviceGet) &&
               entry("cuDeviceGetAttribute", d.DeviceGetAttribute) &&
               entry("cuMulticastCreate", d.MulticastCreate) &&
               entry("cuMulticastGetGranularity", d.MulticastGetGranularity) &&
               entry("cuMulticastAddDevice", d.MulticastAddDevice) &&
               entry("cuMulticastBindMem", d.MulticastBindMem) &&
               entry("cuMulticastUnbind", d.MulticastUnbind) && entry("cuMemCreate", d.MemCreate) &&
               entry("cuMemRelease", d.MemRelease) &&
               entry("cuMemGetAllocationGranularity", d.MemGetAllocationGranularity) &&
               entry("cuMemAddressReserve", d.MemAddressReserve) &&
               entry("cuMemAddressFree", d.MemAddressFree) && entry("cuMemMap", d.MemMap) &&
               entry("cuMemUnmap", d.MemUnmap) && entry("cuMemSetAccess", d.MemSetAccess) &&
               entry("cuMemExportToShareableHandle", d.MemExportToShareableHandle) &&
               entry("cuMemImportFromShareableHandle", d.MemImportFromShareableHandle);
    });
    return d;
}

prngd_status cu_fail(CUresult r, const char *what) {
    const char *s = "?";
    if (drv().GetErrorString) drv().GetErrorString(r, &s);
    return mc_fail(PRNGD_ECUDA, "%s: %s (CUresult %d)", what, s, (int)r);
}

}  // namespace

// One rank's view of the multicast accumulator.
struct prngd_mc {
    CUmemGenericAllocationHandle mc = 0;    // multicast object (imported on ranks != owner)
    CUmemGenericAllocationHandle phys = 0;  // this rank's physical copy
    CUdeviceptr mc_va = 0, uc_va = 0;       // multicast / unicast mappings
    size_t bytes = 0;                       // rounded to the multicast granularity
    CUdevice dev = 0;
    int export_fd = -1;
    bool bound = false;
};

extern "C" {

PRNGD_API prngd_status prngd_mc_supported(int *supported) {
    if (!supported) return mc_fail(PRNGD_EINVAL, "null argument");
    *supported = 0;
    const Drv &d = drv();
    if (!d.ok) return PRNGD_OK;  // driver without the multicast API: not supported
    int ord = 0;
    if (cudaGetDevice(&ord) != cudaSuccess) return mc_fail(PRNGD_ECUDA, "cudaGetDevice failed");
    CUdevice dev;
    CUresult r = d.DeviceGet(&dev, ord);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuDeviceGet");
    int v = 0;
    r = d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuDeviceGetAttribute(MULTICAST_SUPPORTED)");
    *supported = v;
    return PRNGD_OK;
}

PRNGD_API prngd_status prngd_mc_create(uint64_t bytes, uint32_t n_devices, prngd_mc **out,
                                       int *export_fd) {
    if (!out || !export_fd || bytes == 0 || n_devices == 0)
        return mc_fail(PRNGD_EINVAL, "null argument or zero size / devices");
    *out = nullptr;
    *export_fd = -1;
    const Drv &d = drv();
    if (!d.ok) return mc_fail(PRNGD_EUNSUPPORTED, "driver has no multicast entry points");
    CUmulticastObjectProp prop;
    std::memset(&prop, 0, sizeof(prop));
    prop.numDevices = n_devices;
    prop.size = bytes;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CUresult r = d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMulticastGetGranularity");
    prop.size = (bytes + gran - 1) / gran * gran;
    prngd_mc *m = new (std::nothrow) prngd_mc();
    if (!m) return mc_fail(PRNGD_ENOMEM, "host allocation");
    m->bytes = prop.size;
    r = d.MulticastCreate(&m->mc, &prop);
    if (r != CUDA_SUCCESS) {
        delete m;
        return cu_fail(r, "cuMulticastCreate");
    }
    int fd = -1;
    r = d.MemExportToShareableHandle(&fd, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) {
        d.MemRelease(m->mc);
        delete m;
        return cu_fail(r, "cuMemExportToShareableHandle");
    }
    // let the other ranks' processes fetch the descriptor with pidfd_getfd (Yama ptrace scope)
    prctl(PR_SET_PTRACER, PR_SET_PTRACER_ANY, 0, 0, 0);
    m->export_fd = fd;
    *export_fd = fd;
    *out = m;
    return PRNGD_OK;
}

PRNGD_API prngd_status prngd_mc_import(int owner_pid, int owner_fd, uint64_t bytes, prngd_mc **out) {
    if (!out || bytes == 0) return mc_fail(PRNGD_EINVAL, "null argument or zero size");
    *out = nullptr;
    const Drv &d = drv();
    if (!d.ok) return mc_fail(PRNGD_EUNSUPPORTED, "driver has no multicast entry points");
    const long pidfd = syscall(SYS_pidfd_open, (pid_t)owner_pid, 0);
    if (pidfd < 0) return mc_fail(PRNGD_ECUDA, "pidfd_open(%d): %s", owner_pid, std::strerror(errno));
    const long fd = syscall(SYS_pidfd_getfd, (int)pidfd, owner_fd, 0);
    const int err = errno;
    close((int)pidfd);
    if (fd < 0) return mc_fail(PRNGD_ECUDA, "pidfd_getfd(%d): %s", owner_fd, std::strerror(err));
    prngd_mc *m = new (std::nothrow) prngd_mc();
    if (!m) {
        close((int)fd);
        return mc_fail(PRNGD_ENOMEM, "host allocation");
    }
    CUresult r = d.MemImportFromShareableHandle(&m->mc, (void *)(uintptr_t)fd,
                                                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close((int)fd);
    if (r != CUDA_SUCCESS) {
        delete m;
        return cu_fail(r, "cuMemImportFromShareableHandle");
    }
    m->bytes = bytes;
    *out = m;
    return PRNGD_OK;
}

PRNGD_API uint64_t prngd_mc_bytes(const prngd_mc *m) { return m ? m->bytes : 0; }

// Step 2 (every rank, after the owner created and the others imported): add this process's
// current device.  Every rank must have added its device before any rank binds memory.
PRNGD_API prngd_status prngd_mc_add_device(prngd_mc *m) {
    if (!m) return mc_fail(PRNGD_EINVAL, "null handle");
    const Drv &d = drv();
    int ord = 0;
    if (cudaGetDevice(&ord) != cudaSuccess) return mc_fail(PRNGD_ECUDA, "cudaGetDevice failed");
    CUresult r = d.DeviceGet(&m->dev, ord);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuDeviceGet");
    r = d.MulticastAddDevice(m->mc, m->dev);
    return r == CUDA_SUCCESS ? PRNGD_OK : cu_fail(r, "cuMulticastAddDevice");
}

// Step 3 (every rank, after a barrier that follows step 2): allocate this device's copy, bind
// it to the multicast object, map the multicast address (*mc_ptr: the address the kernels reduce
// through) and the local copy (*local_ptr: where this rank reads the reduced result), zeroed.
PRNGD_API prngd_status prngd_mc_bind_map(prngd_mc *m, void **mc_ptr, void **local_ptr) {
    if (!m || !mc_ptr || !local_ptr) return mc_fail(PRNGD_EINVAL, "null argument");
    const Drv &d = drv();
    if (m->export_fd >= 0) {
        // every rank has imported the descriptor by now (the caller's barrier after step 2):
        // withdraw the ptrace permission prngd_mc_create granted and close the export
        prctl(PR_SET_PTRACER, 0, 0, 0, 0);
        close(m->export_fd);
        m->export_fd = -1;
    }
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = m->dev;
    size_t pg = 0;
    CUresult r = d.MemGetAllocationGranularity(&pg, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemGetAllocationGranularity");
    if (m->bytes % pg) m->bytes = (m->bytes + pg - 1) / pg * pg;
    if ((r = d.MemCreate(&m->phys, m->bytes, &ap, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMemCreate");
    if ((r = d.MulticastBindMem(m->mc, 0, m->phys, 0, m->bytes, 0)) != CUDA_SUCCESS)
        return cu_fail(r, "cuMulticastBindMem");
    m->bound = true;
    CUmemAccessDesc ad;
    std::memset(&ad, 0, sizeof(ad));
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = m->dev;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if ((r = d.MemAddressReserve(&m->uc_va, m->bytes, pg, 0, 0)) != CUDA_SUCCESS ||
        (r = d.MemMap(m->uc_va, m->bytes, 0, m->phys, 0)) != CUDA_SUCCESS ||
        (r = d.MemSetAccess(m->uc_va, m->bytes, &ad, 1)) != CUDA_SUCCESS)
        return cu_fail(r, "map the local copy");
    if ((r = d.MemAddressReserve(&m->mc_va, m->bytes, pg, 0, 0)) != CUDA_SUCCESS ||
        (r = d.MemMap(m->mc_va, m->bytes, 0, m->mc, 0)) != CUDA_SUCCESS ||
        (r = d.MemSetAccess(m->mc_va, m->bytes, &ad, 1)) != CUDA_SUCCESS)
        return cu_fail(r, "map the multicast address");
    if (cudaMemset((void *)m->uc_va, 0, m->bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        return mc_fail(PRNGD_ECUDA, "zeroing the local copy failed");
    *mc_ptr = (void *)m->mc_va;
    *local_ptr = (void *)m->uc_va;
    return PRNGD_OK;
}

PRNGD_API prngd_status prngd_mc_destroy(prngd_mc *m) {
    if (!m) return PRNGD_OK;
    const Drv &d = drv();
    if (d.ok) {
        if (m->mc_va) {
            d.MemUnmap(m->mc_va, m->bytes);
            d.MemAddressFree(m->mc_va, m->bytes);
        }
        if (m->uc_va) {
            d.MemUnmap(m->uc_va, m->bytes);
            d.MemAddressFree(m->uc_va, m->bytes);
        }
        if (m->bound) d.MulticastUnbind(m->mc, m->dev, 0, m->bytes);
        if (m->phys) d.MemRelease(m->phys);
        if (m->mc) d.MemRelease(m->mc);
    }
    if (m->export_fd >= 0) close(m->export_fd);
    delete m;
    return PRNGD_OK;
}

}  // extern "C"
