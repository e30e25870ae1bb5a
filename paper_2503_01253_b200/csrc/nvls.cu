// nvls.cu -- NVLink SHARP (NVLS) multicast C buffers for the column-sharded layer (SURVEY 8(f)1:
// "an NVLS multicast epilogue (multimem.st into a symmetric-memory C) so tiles land on all peers as
// they retire").  A multicast object spans the G ranks' devices; every rank binds its own physical
// buffer to it and maps two views: the multicast address (stores through it reach every bound
// buffer, replicated by the NVSwitch) and the unicast address of its own replica.  The SIMT
// kernel's exchange epilogue then writes each C tile once, with multimem.st, instead of G peer
// stores (nm_spmm_mc).  Collective setup (rank 0 creates and exports a fabric handle, every rank
// imports it and adds its device, then -- after all devices are in -- binds and maps):
//   nm_mc_create -> nm_mc_export -> (exchange) -> nm_mc_import -> nm_mc_add_device -> (barrier)
//   -> nm_mc_bind_map ... nm_mc_free.
// Driver entry points are fetched at run time (cudaGetDriverEntryPoint), as for TMA descriptors.
#include <cuda.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace nm {
namespace {

struct McDrv {
    CUresult (*create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*add_device)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*bind_mem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                         unsigned long long) = nullptr;
    CUresult (*unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*mc_gran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    CUresult (*mem_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*mem_gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*export_h)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
    CUresult (*import_h)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
    CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
    CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*dev_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
    bool ok = false;
};

template <typename F>
static bool entry(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return false;
    }
    fn = reinterpret_cast<F>(p);
    return true;
}

static const McDrv& drv() {
    static McDrv d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = entry("cuMulticastCreate", d.create) && entry("cuMulticastAddDevice", d.add_device) &&
               entry("cuMulticastBindMem", d.bind_mem) && entry("cuMulticastUnbind", d.unbind) &&
               entry("cuMulticastGetGranularity", d.mc_gran) && entry("cuMemCreate", d.mem_create) &&
               entry("cuMemGetAllocationGranularity", d.mem_gran) && entry("cuMemAddressReserve", d.reserve) &&
               entry("cuMemMap", d.map) && entry("cuMemSetAccess", d.set_access) &&
               entry("cuMemExportToShareableHandle", d.export_h) &&
               entry("cuMemImportFromShareableHandle", d.import_h) && entry("cuMemUnmap", d.unmap) &&
               entry("cuMemAddressFree", d.addr_free) && entry("cuMemRelease", d.release) &&
               entry("cuDeviceGetAttribute", d.dev_attr);
    });
    return d;
}

static nm_status cu_fail(CUresult r, const char* what) {
    return fail(NM_ERR_CUDA, std::string(what) + " failed (CUresult " + std::to_string(static_cast<int>(r)) + ")");
}

}  // namespace
}  // namespace nm

using namespace nm;

extern "C" {

nm_status nm_mc_supported(int* supported) {
    if (!supported) return fail(NM_ERR_NULL, "nm_mc_supported: NULL");
    *supported = 0;
    nm_status st = require_device();
    if (st) return st;
    const McDrv& d = drv();
    int v = 0;
    if (d.ok && d.dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, static_cast<CUdevice>(current_device())) !=
                    CUDA_SUCCESS)
        v = 0;
    if (v && d.ok) {
        // the attribute says the device can; a trial object says whether this process may (with one
        // visible GPU of a multi-GPU node cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE)
        CUmulticastObjectProp prop{};
        prop.numDevices = 1;
        size_t gran = 0;
        CUmemGenericAllocationHandle h = 0;
        prop.size = 2u << 20;
        if (d.mc_gran(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && gran > 0) {
            prop.size = (prop.size + gran - 1) / gran * gran;
            if (d.create(&h, &prop) == CUDA_SUCCESS) {
                d.release(h);
                *supported = 1;
            }
        }
    }
    return NM_OK;
}

nm_status nm_mc_create(int64_t bytes, int num_devices, uint64_t* mc, int64_t* mc_bytes) {
    if (!mc || !mc_bytes) return fail(NM_ERR_NULL, "nm_mc_create: NULL");
    if (bytes <= 0 || num_devices < 1 || num_devices > 8) return fail(NM_ERR_SHAPE, "nm_mc_create: bytes > 0, 1..8 devices");
    nm_status st = require_device();
    if (st) return st;
    const McDrv& d = drv();
    if (!d.ok) return fail(NM_ERR_UNSUPPORTED, "nm_mc_create: multicast driver entry points unavailable");
    CUmulticastObjectProp prop{};
    prop.numDevices = static_cast<unsigned>(num_devices);
    prop.handleTypes = num_devices > 1 ? CU_MEM_HANDLE_TYPE_FABRIC : 0;
    prop.size = static_cast<size_t>(bytes);
    size_t gran = 0;
    CUresult r = d.mc_gran(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMulticastGetGranularity");
    prop.size = (static_cast<size_t>(bytes) + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h = 0;
    if ((r = d.create(&h, &prop)) != CUDA_SUCCESS) return cu_fail(r, "cuMulticastCreate");
    *mc = h;
    *mc_bytes = static_cast<int64_t>(prop.size);
    return NM_OK;
}

nm_status nm_mc_export(uint64_t mc, void* fabric_handle) {
    if (!fabric_handle) return fail(NM_ERR_NULL, "nm_mc_export: NULL");
    const McDrv& d = drv();
    if (!d.ok) return fail(NM_ERR_UNSUPPORTED, "multicast unavailable");
    CUmemFabricHandle fh;
    const CUresult r = d.export_h(&fh, mc, CU_MEM_HANDLE_TYPE_FABRIC, 0);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemExportToShareableHandle (fabric)");
    std::memcpy(fabric_handle, &fh, sizeof(fh));
    return NM_OK;
}

nm_status nm_mc_import(const void* fabric_handle, uint64_t* mc) {
    if (!fabric_handle || !mc) return fail(NM_ERR_NULL, "nm_mc_import: NULL");
    const McDrv& d = drv();
    if (!d.ok) return fail(NM_ERR_UNSUPPORTED, "multicast unavailable");
    CUmemFabricHandle fh;
    std::memcpy(&fh, fabric_handle, sizeof(fh));
    CUmemGenericAllocationHandle h = 0;
    const CUresult r = d.import_h(&h, &fh, CU_MEM_HANDLE_TYPE_FABRIC);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemImportFromShareableHandle (fabric)");
    *mc = h;
    return NM_OK;
}

nm_status nm_mc_add_device(uint64_t mc) {
    const McDrv& d = drv();
    if (!d.ok) return fail(NM_ERR_UNSUPPORTED, "multicast unavailable");
    const CUresult r = d.add_device(mc, static_cast<CUdevice>(current_device()));
    return r == CUDA_SUCCESS ? NM_OK : cu_fail(r, "cuMulticastAddDevice");
}

nm_status nm_mc_bind_map(uint64_t mc, int64_t mc_bytes, uint64_t* mem, void** uc_ptr, void** mc_ptr) {
    if (!mem || !uc_ptr || !mc_ptr) return fail(NM_ERR_NULL, "nm_mc_bind_map: NULL");
    const McDrv& d = drv();
    if (!d.ok) return fail(NM_ERR_UNSUPPORTED, "multicast unavailable");
    const int dev = current_device();
    const size_t size = static_cast<size_t>(mc_bytes);
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev;
    CUmemGenericAllocationHandle h = 0;
    CUresult r = d.mem_create(&h, size, &prop, 0);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemCreate");
    if ((r = d.bind_mem(mc, 0, h, 0, size, 0)) != CUDA_SUCCESS) {
        d.release(h);
        return cu_fail(r, "cuMulticastBindMem");
    }
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr uc = 0, mcp = 0;
    if ((r = d.reserve(&uc, size, 0, 0, 0)) != CUDA_SUCCESS || (r = d.map(uc, size, 0, h, 0)) != CUDA_SUCCESS ||
        (r = d.set_access(uc, size, &acc, 1)) != CUDA_SUCCESS || (r = d.reserve(&mcp, size, 0, 0, 0)) != CUDA_SUCCESS ||
        (r = d.map(mcp, size, 0, mc, 0)) != CUDA_SUCCESS || (r = d.set_access(mcp, size, &acc, 1)) != CUDA_SUCCESS)
        return cu_fail(r, "nm_mc_bind_map: reserve / map / set access");
    *mem = h;
    *uc_ptr = reinterpret_cast<void*>(uc);
    *mc_ptr = reinterpret_cast<void*>(mcp);
    return NM_OK;
}

nm_status nm_mc_free(uint64_t mc, uint64_t mem, void* uc_ptr, void* mc_ptr, int64_t mc_bytes) {
    const McDrv& d = drv();
    if (!d.ok) return fail(NM_ERR_UNSUPPORTED, "multicast unavailable");
    const size_t size = static_cast<size_t>(mc_bytes);
    cudaDeviceSynchronize();
    if (mc_ptr) {
        d.unmap(reinterpret_cast<CUdeviceptr>(mc_ptr), size);
        d.addr_free(reinterpret_cast<CUdeviceptr>(mc_ptr), size);
    }
    if (uc_ptr) {
        d.unmap(reinterpret_cast<CUdeviceptr>(uc_ptr), size);
        d.addr_free(reinterpret_cast<CUdeviceptr>(uc_ptr), size);
    }
    if (mem) {
        d.unbind(mc, static_cast<CUdevice>(current_device()), 0, size);
        d.release(mem);
    }
    if (mc) d.release(mc);
    return NM_OK;
}

}  // extern "C"
