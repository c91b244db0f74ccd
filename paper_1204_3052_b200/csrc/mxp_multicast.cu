// NVLS multicast buffers for the fused row-sharded exchange (SURVEY §5
// stretch, §8(e)): one multicast object per shared buffer group, every rank
// binds its own device memory to it, and a store to the multicast address is
// written by the NVSwitch into every rank's copy — each output tile leaves
// its GPU once instead of once per peer (the peer-store exchange,
// mxp_gemm_rows_planes_peers, writes it N-1 times over NVLink).
//
// Driver API through the runtime's entry-point query (the library does not
// link libcuda).  The creator exports a FABRIC handle (64 opaque bytes) that
// the other ranks import; binding happens after every rank has added its
// device (cuMulticastBindMem requires the full team).
#include <cstring>
#include <new>

#include "../../include/matexpo_b200.h"
#include "mxp_internal.h"

struct mxp_mc_s {
    int device = 0;
    CUdevice cudev = 0;
    size_t size = 0;
    CUmemGenericAllocationHandle mc = 0, phys = 0;
    CUdeviceptr uc_va = 0, mc_va = 0;
    bool have_mc = false, have_phys = false, bound = false, uc_mapped = false, mc_mapped = false;
};

// defined in mxp_api.cu: the library's error slot and a handle's device
int mxp_internal_fail(int code, const char* fmt, ...);
int mxp_internal_device(mxp_handle h);

namespace {

struct DrvApi {
    CUresult (*deviceGet)(CUdevice*, int) = nullptr;
    CUresult (*deviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
    CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t,
                          size_t, unsigned long long) = nullptr;
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*mcGetGranularity)(size_t*, const CUmulticastObjectProp*,
                                 CUmulticastGranularity_flags) = nullptr;
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                          unsigned long long) = nullptr;
    CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*memAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*memAddressFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*memGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                            CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                          unsigned long long) = nullptr;
    CUresult (*memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
    bool ok = false;
};

template <typename F>
bool sym(F& fn, const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
        return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

const DrvApi& drv() {
    static DrvApi d = [] {
        DrvApi a;
        a.ok = sym(a.deviceGet, "cuDeviceGet") && sym(a.deviceGetAttribute, "cuDeviceGetAttribute") &&
               sym(a.mcCreate, "cuMulticastCreate") && sym(a.mcAddDevice, "cuMulticastAddDevice") &&
               sym(a.mcBindMem, "cuMulticastBindMem") && sym(a.mcUnbind, "cuMulticastUnbind") &&
               sym(a.mcGetGranularity, "cuMulticastGetGranularity") &&
               sym(a.memCreate, "cuMemCreate") && sym(a.memRelease, "cuMemRelease") &&
               sym(a.memAddressReserve, "cuMemAddressReserve") &&
               sym(a.memAddressFree, "cuMemAddressFree") && sym(a.memMap, "cuMemMap") &&
               sym(a.memUnmap, "cuMemUnmap") && sym(a.memSetAccess, "cuMemSetAccess") &&
               sym(a.memGetAllocationGranularity, "cuMemGetAllocationGranularity") &&
               sym(a.memExport, "cuMemExportToShareableHandle") &&
               sym(a.memImport, "cuMemImportFromShareableHandle");
        return a;
    }();
    return d;
}

int drv_fail(CUresult r, const char* what) {
    return mxp_internal_fail(MXP_E_CUDA, "%s failed (CUresult %d)", what, static_cast<int>(r));
}

#define MXP_DRV(expr, what)                                  \
    do {                                                     \
        CUresult _r = (expr);                                \
        if (_r != CUDA_SUCCESS) return drv_fail(_r, what);   \
    } while (0)

size_t round_up_sz(size_t x, size_t m) { return (x + m - 1) / m * m; }

int mc_prop(int nranks, size_t bytes, CUmulticastObjectProp* prop) {
    std::memset(prop, 0, sizeof *prop);
    prop->numDevices = static_cast<unsigned>(nranks);
    prop->handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    prop->size = bytes;
    size_t gran = 0;
    MXP_DRV(drv().mcGetGranularity(&gran, prop, CU_MULTICAST_GRANULARITY_RECOMMENDED),
            "cuMulticastGetGranularity");
    prop->size = round_up_sz(bytes, gran);
    return MXP_OK;
}

}  // namespace

extern "C" {

int mxp_mc_supported(mxp_handle h, int* ok) {
    if (!h || !ok) return mxp_internal_fail(MXP_E_VALIDATION, "null argument");
    *ok = 0;
    const DrvApi& d = drv();
    if (!d.ok) return MXP_OK;
    int dev = mxp_internal_device(h);
    CUdevice cd;
    if (d.deviceGet(&cd, dev) != CUDA_SUCCESS) return MXP_OK;
    int mc = 0, fab = 0;
    d.deviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd);
    d.deviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, cd);
    *ok = (mc && fab) ? 1 : 0;
    return MXP_OK;
}

int mxp_mc_create(mxp_handle h, int nranks, size_t bytes, void* handle_out, mxp_mc* out) {
    if (!h || !handle_out || !out || nranks < 1 || bytes == 0)
        return mxp_internal_fail(MXP_E_VALIDATION, "bad multicast create arguments");
    *out = nullptr;
    if (!drv().ok) return mxp_internal_fail(MXP_E_UNSUPPORTED, "driver lacks the multicast API");
    cudaSetDevice(mxp_internal_device(h));
    auto* m = new (std::nothrow) mxp_mc_s();
    if (!m) return mxp_internal_fail(MXP_E_CUDA, "out of host memory");
    m->device = mxp_internal_device(h);
    CUmulticastObjectProp prop;
    int rc = mc_prop(nranks, bytes, &prop);
    if (rc) {
        delete m;
        return rc;
    }
    m->size = prop.size;
    CUresult r = drv().deviceGet(&m->cudev, m->device);
    if (r == CUDA_SUCCESS) r = drv().mcCreate(&m->mc, &prop);
    if (r != CUDA_SUCCESS) {
        delete m;
        return drv_fail(r, "cuMulticastCreate");
    }
    m->have_mc = true;
    r = drv().memExport(handle_out, m->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0);
    if (r == CUDA_SUCCESS) r = drv().mcAddDevice(m->mc, m->cudev);
    if (r != CUDA_SUCCESS) {
        mxp_mc_destroy(m);
        return drv_fail(r, "multicast export / add device");
    }
    *out = m;
    return MXP_OK;
}

int mxp_mc_import(mxp_handle h, const void* handle, size_t bytes, mxp_mc* out) {
    if (!h || !handle || !out || bytes == 0)
        return mxp_internal_fail(MXP_E_VALIDATION, "bad multicast import arguments");
    *out = nullptr;
    if (!drv().ok) return mxp_internal_fail(MXP_E_UNSUPPORTED, "driver lacks the multicast API");
    cudaSetDevice(mxp_internal_device(h));
    auto* m = new (std::nothrow) mxp_mc_s();
    if (!m) return mxp_internal_fail(MXP_E_CUDA, "out of host memory");
    m->device = mxp_internal_device(h);
    m->size = bytes;
    CUmemFabricHandle fh;
    std::memcpy(&fh, handle, sizeof fh);
    CUresult r = drv().deviceGet(&m->cudev, m->device);
    if (r == CUDA_SUCCESS) r = drv().memImport(&m->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC);
    if (r != CUDA_SUCCESS) {
        delete m;
        return drv_fail(r, "cuMemImportFromShareableHandle (multicast)");
    }
    m->have_mc = true;
    r = drv().mcAddDevice(m->mc, m->cudev);
    if (r != CUDA_SUCCESS) {
        mxp_mc_destroy(m);
        return drv_fail(r, "cuMulticastAddDevice");
    }
    *out = m;
    return MXP_OK;
}

int mxp_mc_size(mxp_mc m, size_t* bytes) {
    if (!m || !bytes) return mxp_internal_fail(MXP_E_VALIDATION, "null argument");
    *bytes = m->size;
    return MXP_OK;
}

int mxp_mc_bind(mxp_mc m, void** local_ptr, void** mc_ptr) {
    if (!m || !local_ptr || !mc_ptr) return mxp_internal_fail(MXP_E_VALIDATION, "null argument");
    const DrvApi& d = drv();
    cudaSetDevice(m->device);
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof ap);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = m->device;
    size_t gran = 0;
    MXP_DRV(d.memGetAllocationGranularity(&gran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
            "cuMemGetAllocationGranularity");
    m->size = round_up_sz(m->size, gran);
    MXP_DRV(d.memCreate(&m->phys, m->size, &ap, 0), "cuMemCreate");
    m->have_phys = true;
    MXP_DRV(d.mcBindMem(m->mc, 0, m->phys, 0, m->size, 0), "cuMulticastBindMem");
    m->bound = true;
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof acc);
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = m->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    MXP_DRV(d.memAddressReserve(&m->uc_va, m->size, gran, 0, 0), "cuMemAddressReserve");
    MXP_DRV(d.memMap(m->uc_va, m->size, 0, m->phys, 0), "cuMemMap (unicast)");
    m->uc_mapped = true;
    MXP_DRV(d.memSetAccess(m->uc_va, m->size, &acc, 1), "cuMemSetAccess (unicast)");
    MXP_DRV(d.memAddressReserve(&m->mc_va, m->size, gran, 0, 0), "cuMemAddressReserve");
    MXP_DRV(d.memMap(m->mc_va, m->size, 0, m->mc, 0), "cuMemMap (multicast)");
    m->mc_mapped = true;
    MXP_DRV(d.memSetAccess(m->mc_va, m->size, &acc, 1), "cuMemSetAccess (multicast)");
    *local_ptr = reinterpret_cast<void*>(m->uc_va);
    *mc_ptr = reinterpret_cast<void*>(m->mc_va);
    return MXP_OK;
}

int mxp_mc_destroy(mxp_mc m) {
    if (!m) return MXP_OK;
    const DrvApi& d = drv();
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    if (m->mc_mapped) d.memUnmap(m->mc_va, m->size);
    if (m->mc_va) d.memAddressFree(m->mc_va, m->size);
    if (m->uc_mapped) d.memUnmap(m->uc_va, m->size);
    if (m->uc_va) d.memAddressFree(m->uc_va, m->size);
    if (m->bound) d.mcUnbind(m->mc, m->cudev, 0, m->size);
    if (m->have_phys) d.memRelease(m->phys);
    if (m->have_mc) d.memRelease(m->mc);
    delete m;
    return MXP_OK;
}

}  // extern "C"
