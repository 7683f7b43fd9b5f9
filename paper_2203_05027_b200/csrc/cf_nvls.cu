// NVLink SHARP (NVLS) stage of the row-sharded step (SURVEY §2 K7 stage 2, §8e "Fused NVLS
// kernel"): the exchange of the row-sharded iteration done by the NVSwitch itself.
//
//   partial A_r^T h_r  --(each rank writes its own copy of one multicast buffer)-->
//   multimem.ld_reduce.add.f64 on the multicast address: the switch returns the SUM over
//   every rank's copy -> column update on the rank's slice (x_update, z_update, delta)
//   -> multimem.st.f64 of x+ on the multicast x buffer: the switch writes it into every
//   rank's replica.
//
// One kernel replaces reduce-scatter + cf_column_update + all-gather, like the P2P step
// (cf_column_update_p2p), but each value crosses NVLink once in each direction whatever
// the world size. The cross-rank ordering (partials written before any rank reduces,
// replicas filled before any rank's row pass) is a device-side flag barrier on a
// multicast counter (multimem.red.release + ld.acquire spin), not a host round trip.
//
// Multicast objects come from the CUDA driver's VMM API (cuMulticastCreate, one physical
// allocation per rank bound to it, unicast + multicast mappings). The driver entry points
// are fetched with cudaGetDriverEntryPoint, so libcfb200 does not link libcuda. For
// world > 1 the creating rank exports a POSIX file descriptor that the others import
// (the Python driver passes it over a Unix socket). The sum order inside the switch is
// the hardware's: bit-identical to the rank-order sum for 1 or 2 ranks (a + b == b + a),
// equal to rounding beyond.
#include <cuda.h>

#include "cf_common.h"

struct cf_mc {
    CUmemGenericAllocationHandle mc_handle = 0;
    CUmemGenericAllocationHandle mem_handle = 0;
    CUdeviceptr uc = 0, mcva = 0;
    size_t size = 0;
    int dev = -1;
    bool added = false, bound = false;
};

namespace cf {
namespace {

struct Drv {
    decltype(&cuMulticastCreate) mc_create = nullptr;
    decltype(&cuMulticastAddDevice) mc_add = nullptr;
    decltype(&cuMulticastBindMem) mc_bind = nullptr;
    decltype(&cuMulticastUnbind) mc_unbind = nullptr;
    decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
    decltype(&cuMemCreate) mem_create = nullptr;
    decltype(&cuMemRelease) mem_release = nullptr;
    decltype(&cuMemAddressReserve) va_reserve = nullptr;
    decltype(&cuMemAddressFree) va_free = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemExportToShareableHandle) export_h = nullptr;
    decltype(&cuMemImportFromShareableHandle) import_h = nullptr;
    decltype(&cuDeviceGetAttribute) dev_attr = nullptr;
    decltype(&cuMemGetAllocationGranularity) mem_gran = nullptr;
    bool ok = false;
};

const Drv& drv() {
    static const Drv d = [] {
        Drv x;
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn;
        };
        x.ok = get("cuMulticastCreate", (void**)&x.mc_create) && get("cuMulticastAddDevice", (void**)&x.mc_add) &&
               get("cuMulticastBindMem", (void**)&x.mc_bind) && get("cuMulticastUnbind", (void**)&x.mc_unbind) &&
               get("cuMulticastGetGranularity", (void**)&x.mc_gran) && get("cuMemCreate", (void**)&x.mem_create) &&
               get("cuMemRelease", (void**)&x.mem_release) && get("cuMemAddressReserve", (void**)&x.va_reserve) &&
               get("cuMemAddressFree", (void**)&x.va_free) && get("cuMemMap", (void**)&x.map) &&
               get("cuMemUnmap", (void**)&x.unmap) && get("cuMemSetAccess", (void**)&x.set_access) &&
               get("cuMemExportToShareableHandle", (void**)&x.export_h) &&
               get("cuMemImportFromShareableHandle", (void**)&x.import_h) &&
               get("cuDeviceGetAttribute", (void**)&x.dev_attr) &&
               get("cuMemGetAllocationGranularity", (void**)&x.mem_gran);
        cudaGetLastError();
        return x;
    }();
    return d;
}

int drv_fail(CUresult r, const char* what) {
    set_error(std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
    return CF_ECUDA;
}
#define CF_CU(call, what)                            \
    do {                                             \
        CUresult _r = (call);                        \
        if (_r != CUDA_SUCCESS) return drv_fail(_r, what); \
    } while (0)

int need_drv() {
    if (!drv().ok) {
        set_error("CUDA driver multicast entry points unavailable");
        return CF_ECUDA;
    }
    return CF_OK;
}

CUmulticastObjectProp mc_prop(size_t size, int world) {
    CUmulticastObjectProp p{};
    p.numDevices = (unsigned)world;
    p.size = size;
    p.handleTypes = world > 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
    return p;
}

// ---------------------------------------------------------------- kernels
__device__ __forceinline__ double mc_ld_reduce_add(const double* mc) {
    double v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc) : "memory");
    return v;
}
__device__ __forceinline__ void mc_st(double* mc, double v) {
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mc), "d"(v) : "memory");
}

// cf_column_update_p2p with the reduce and the broadcast done by the switch
__global__ void k_col_update_nvls(int64_t n, const double* parts_mc, const double* cnt, const double* c, double* x,
                                  double* z, double* delta, double mu, const int32_t* cone_ptr, double* wbuf,
                                  double* x_mc) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double ath = mc_ld_reduce_add(parts_mc + j);
        const double cj = cnt[j];
        const double fv = 1.0 / (1.0 + cj);
        const double xj = x[j], zj = z[j], dj = delta[j];
        const double dm = dj / mu;
        const double v = __dadd_rn(__dmul_rn(cj, xj), ath);
        const double xp = fv * (((v + zj) + dm) - c[j] / mu);
        const double w = xp - dm;
        x[j] = xp;
        if (x_mc) mc_st(x_mc + j, xp);
        if (!cone_ptr) {
            const double zp = w > 0.0 ? w : 0.0;
            z[j] = zp;
            delta[j] = dj + mu * (zp - xp);
        } else {
            wbuf[j] = w;
        }
    }
    asm volatile("fence.sc.sys;" ::: "memory");   // multimem stores performed before the barrier's release
}

__global__ void k_cone_update_nvls(int64_t n_blocks, const int32_t* cone_ptr, const double* wbuf, const double* x,
                                   double* z, double* delta, double mu) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_blocks;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int off = cone_ptr[q], size = cone_ptr[q + 1] - off;
        const double w0 = wbuf[off];
        double ssq = 0.0;
        for (int t = 1; t < size; ++t) ssq = __dadd_rn(ssq, __dmul_rn(wbuf[off + t], wbuf[off + t]));
        const double alpha = sqrt(ssq);
        for (int t = 0; t < size; ++t) {
            double zt;
            if (alpha <= -w0) {
                zt = 0.0;
            } else if (alpha <= w0) {
                zt = wbuf[off + t];
            } else if (t == 0) {
                zt = __dadd_rn(__dmul_rn(0.5, w0), __dmul_rn(0.5, alpha));
            } else {
                const double factor = w0 / (2.0 * alpha);
                zt = __dadd_rn(__dmul_rn(0.5, wbuf[off + t]), __dmul_rn(factor, wbuf[off + t]));
            }
            z[off + t] = zt;
            delta[off + t] = delta[off + t] + mu * (zt - x[off + t]);
        }
    }
}

// device-side barrier over the multicast team: every rank adds 1 to the counter in every
// rank's copy (one multimem.red), then waits until its own copy reaches world * epoch
__global__ void k_mc_barrier(uint32_t* flag_mc, const uint32_t* flag_uc, uint32_t target) {
    asm volatile("fence.sc.sys;" ::: "memory");
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(flag_mc), "r"(1u) : "memory");
    uint32_t v = 0;
    do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag_uc) : "memory");
    } while ((int32_t)(v - target) < 0);
}

}  // namespace
}  // namespace cf

using namespace cf;

extern "C" {

int cf_mc_supported(int* supported) {
    if (!supported) return CF_EINVAL;
    *supported = 0;
    if (!drv().ok) return CF_OK;
    int dev = 0;
    CF_CUDA(cudaGetDevice(&dev));
    int v = 0;
    CF_CU(drv().dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)dev), "cuDeviceGetAttribute");
    *supported = v;
    return CF_OK;
}

int cf_mc_create(int64_t bytes, int32_t world, cf_mc** out, int* fd_out) {
    if (!out || bytes <= 0 || world < 1 || (world > 1 && !fd_out)) {
        set_error("cf_mc_create: bad arguments");
        return CF_EINVAL;
    }
    CF_TRY(need_drv());
    *out = nullptr;
    size_t gran = 0;
    CUmulticastObjectProp prop = mc_prop((size_t)bytes, world);
    CF_CU(drv().mc_gran(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    prop.size = ((size_t)bytes + gran - 1) / gran * gran;
    auto* m = new cf_mc();
    m->size = prop.size;
    CUresult r = drv().mc_create(&m->mc_handle, &prop);
    if (r != CUDA_SUCCESS) {
        delete m;
        return drv_fail(r, "cuMulticastCreate");
    }
    if (world > 1) {
        int fd = -1;
        r = drv().export_h(&fd, m->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
        if (r != CUDA_SUCCESS) {
            drv().mem_release(m->mc_handle);
            delete m;
            return drv_fail(r, "cuMemExportToShareableHandle");
        }
        *fd_out = fd;
    }
    *out = m;
    return CF_OK;
}

int cf_mc_import(int fd, int64_t bytes, int32_t world, cf_mc** out) {
    if (!out || bytes <= 0 || world < 2 || fd < 0) {
        set_error("cf_mc_import: bad arguments");
        return CF_EINVAL;
    }
    CF_TRY(need_drv());
    size_t gran = 0;
    CUmulticastObjectProp prop = mc_prop((size_t)bytes, world);
    CF_CU(drv().mc_gran(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    auto* m = new cf_mc();
    m->size = ((size_t)bytes + gran - 1) / gran * gran;
    CUresult r = drv().import_h(&m->mc_handle, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) {
        delete m;
        return drv_fail(r, "cuMemImportFromShareableHandle");
    }
    *out = m;
    return CF_OK;
}

int cf_mc_add_device(cf_mc* m) {
    if (!m) return CF_EINVAL;
    CF_TRY(need_drv());
    CF_CUDA(cudaGetDevice(&m->dev));
    CF_CU(drv().mc_add(m->mc_handle, (CUdevice)m->dev), "cuMulticastAddDevice");
    m->added = true;
    return CF_OK;
}

// Bind this rank's physical memory (zeroed) and map the unicast and multicast views.
// Blocks until every rank of the team has called cf_mc_add_device.
int cf_mc_bind(cf_mc* m, void** uc_ptr, void** mc_ptr) {
    if (!m || !m->added || !uc_ptr || !mc_ptr) {
        set_error("cf_mc_bind: create/import and add the device first");
        return CF_EINVAL;
    }
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = m->dev;
    size_t g = 0;
    CF_CU(drv().mem_gran(&g, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    if (m->size % g) m->size = (m->size + g - 1) / g * g;
    CF_CU(drv().mem_create(&m->mem_handle, m->size, &ap, 0), "cuMemCreate");
    CF_CU(drv().mc_bind(m->mc_handle, 0, m->mem_handle, 0, m->size, 0), "cuMulticastBindMem");
    m->bound = true;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = m->dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CF_CU(drv().va_reserve(&m->uc, m->size, 0, 0, 0), "cuMemAddressReserve");
    CF_CU(drv().map(m->uc, m->size, 0, m->mem_handle, 0), "cuMemMap (unicast)");
    CF_CU(drv().set_access(m->uc, m->size, &acc, 1), "cuMemSetAccess (unicast)");
    CF_CU(drv().va_reserve(&m->mcva, m->size, 0, 0, 0), "cuMemAddressReserve");
    CF_CU(drv().map(m->mcva, m->size, 0, m->mc_handle, 0), "cuMemMap (multicast)");
    CF_CU(drv().set_access(m->mcva, m->size, &acc, 1), "cuMemSetAccess (multicast)");
    CF_CUDA(cudaMemset((void*)m->uc, 0, m->size));
    CF_CUDA(cudaDeviceSynchronize());
    *uc_ptr = (void*)m->uc;
    *mc_ptr = (void*)m->mcva;
    return CF_OK;
}

int cf_mc_destroy(cf_mc* m) {
    if (!m) return CF_OK;
    cudaDeviceSynchronize();
    if (drv().ok) {
        if (m->mcva) {
            drv().unmap(m->mcva, m->size);
            drv().va_free(m->mcva, m->size);
        }
        if (m->uc) {
            drv().unmap(m->uc, m->size);
            drv().va_free(m->uc, m->size);
        }
        if (m->bound) drv().mc_unbind(m->mc_handle, (CUdevice)m->dev, 0, m->size);
        if (m->mem_handle) drv().mem_release(m->mem_handle);
        if (m->mc_handle) drv().mem_release(m->mc_handle);
    }
    delete m;
    return CF_OK;
}

int cf_column_update_nvls(int64_t n, const double* parts_mc, const double* cnt, const double* c, double* x, double* z,
                          double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr, double* x_mc,
                          void* stream) {
    if (n < 0 || (n > 0 && (!parts_mc || !cnt || !c || !x || !z || !delta)) || !(mu > 0.0)) {
        set_error("cf_column_update_nvls: bad arguments");
        return CF_EINVAL;
    }
    if (n == 0) return CF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf<double> w;
    if (cone_ptr) CF_TRY(w.alloc(n));
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_col_update_nvls<<<grid, 256, 0, st>>>(n, parts_mc, cnt, c, x, z, delta, mu, cone_ptr, w.p, x_mc);
    CF_LAUNCHED();
    if (cone_ptr) {
        k_cone_update_nvls<<<(int)std::min<int64_t>((n_blocks + 127) / 128, 148 * 16), 128, 0, st>>>(
            n_blocks, cone_ptr, w.p, x, z, delta, mu);
        CF_LAUNCHED();
        CF_CUDA(cudaStreamSynchronize(st));   // w is released at return
    }
    return CF_OK;
}

int cf_mc_barrier(uint32_t* flag_mc, const uint32_t* flag_uc, uint32_t target, void* stream) {
    if (!flag_mc || !flag_uc) {
        set_error("cf_mc_barrier: NULL flag");
        return CF_EINVAL;
    }
    k_mc_barrier<<<1, 1, 0, (cudaStream_t)stream>>>(flag_mc, flag_uc, target);
    CF_LAUNCHED();
    return CF_OK;
}

}  // extern "C"
