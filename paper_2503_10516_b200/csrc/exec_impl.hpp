// Private declarations shared by the executor's translation units
// (exec.cu, exec_copy.cu, exec_kernel.cu, exec_coll.cu, exec_vnode.cu).
#pragma once

#include "exec.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>
#include <nccl.h>

#include "../../include/cel.h"

namespace cel {

Box map_access(const Mapper& m, const Box& chunk, const Box& ext);  // sched.cpp

namespace detail {
// Driver-API entry points resolved through the runtime (no link-time libcuda
// dependency, so the library also loads on a host without a driver for the
// execute=0 scheduling mode).
struct Drv {
    CUresult (*wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
    CUresult (*write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
    CUresult (*errstr)(CUresult, const char**) = nullptr;
    CUresult (*devattr)(int*, CUdevice_attribute, CUdevice) = nullptr;
    // virtual memory management (in-place growth by mapping)
    CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
    CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
    // multicast objects (NVLS all-gather)
    CUresult (*mc_create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*mc_add_device)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*mc_bind_mem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                            unsigned long long) = nullptr;
    CUresult (*mc_unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*mc_granularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    bool loaded = false;
    bool vmm() const { return reserve && addr_free && create && release && map && unmap && set_access && granularity; }
    bool multicast() const { return vmm() && mc_create && mc_add_device && mc_bind_mem && mc_unbind && mc_granularity; }
    void load() {
        if (loaded) return;
        loaded = true;
        cudaDriverEntryPointQueryResult q;
        auto get = [&](const char* name, auto** fn) {
            cudaGetDriverEntryPoint(name, reinterpret_cast<void**>(fn), cudaEnableDefault, &q);
            if (q != cudaDriverEntryPointSuccess) *fn = nullptr;
        };
        get("cuMemAddressReserve", &reserve);
        get("cuMemAddressFree", &addr_free);
        get("cuMemCreate", &create);
        get("cuMemRelease", &release);
        get("cuMemMap", &map);
        get("cuMemUnmap", &unmap);
        get("cuMemSetAccess", &set_access);
        get("cuMemGetAllocationGranularity", &granularity);
        get("cuMulticastCreate", &mc_create);
        get("cuMulticastAddDevice", &mc_add_device);
        get("cuMulticastBindMem", &mc_bind_mem);
        get("cuMulticastUnbind", &mc_unbind);
        get("cuMulticastGetGranularity", &mc_granularity);
        cudaGetDriverEntryPoint("cuStreamWaitValue64", reinterpret_cast<void**>(&wait64), cudaEnableDefault, &q);
        cudaGetDriverEntryPoint("cuStreamWriteValue64", reinterpret_cast<void**>(&write64), cudaEnableDefault, &q);
        cudaGetDriverEntryPoint("cuGetErrorString", reinterpret_cast<void**>(&errstr), cudaEnableDefault, &q);
        cudaGetDriverEntryPoint("cuDeviceGetAttribute", reinterpret_cast<void**>(&devattr), cudaEnableDefault, &q);
    }
};
inline Drv g_drv;

// NCCL, opened at run time (the process may already hold torch's copy of
// libnccl.so.2; the C API is stable across the 2.2x releases in this image).
struct Nccl {
    ncclResult_t (*get_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allgather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errstr)(ncclResult_t) = nullptr;
    int state = 0;   // 0 not tried, 1 loaded, -1 unavailable
    bool load() {
        if (state) return state > 0;
        state = -1;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        get_id = reinterpret_cast<decltype(get_id)>(dlsym(h, "ncclGetUniqueId"));
        init_rank = reinterpret_cast<decltype(init_rank)>(dlsym(h, "ncclCommInitRank"));
        init_all = reinterpret_cast<decltype(init_all)>(dlsym(h, "ncclCommInitAll"));
        destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "ncclCommDestroy"));
        group_start = reinterpret_cast<decltype(group_start)>(dlsym(h, "ncclGroupStart"));
        group_end = reinterpret_cast<decltype(group_end)>(dlsym(h, "ncclGroupEnd"));
        bcast = reinterpret_cast<decltype(bcast)>(dlsym(h, "ncclBroadcast"));
        allgather = reinterpret_cast<decltype(allgather)>(dlsym(h, "ncclAllGather"));
        errstr = reinterpret_cast<decltype(errstr)>(dlsym(h, "ncclGetErrorString"));
        if (get_id && init_rank && init_all && destroy && group_start && group_end && bcast && errstr) state = 1;
        return state > 0;
    }
};
inline Nccl g_nccl;

inline uint64_t now_ns() {
    return uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now().time_since_epoch())
                        .count());
}

constexpr int kStreamsPerDev = 11;
// work streams 0..4; 5 = eager horizon / epoch flags; 6..10 = flags released
// by an event of work stream (k - 6), so each flag stream's FIFO order follows
// its source stream's completion order (no head-of-line blocking between a
// long-complete flag and one waiting for recent work)
enum { S_COMPUTE = 0, S_COPY = 1, S_PUSH = 2, S_SYNC = 3, S_HALO = 4, S_HSIG = 5, S_SIG0 = 6 };
constexpr int kNumSigStreams = kStreamsPerDev - S_SIG0;   // one per work stream 0..4
constexpr uint64_t kAlign = 512;
inline uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }
}  // namespace detail
using namespace detail;
}  // namespace cel
