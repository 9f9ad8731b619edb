// nvls.cuh -- the data-parallel gradient exchange fused with the update over
// NVLink SHARP: NVSwitch multicast memory instead of an NCCL
// allreduce followed by a separate update pass.
//
// The network arena's [params | grads | velocities] regions (equal layouts,
// abi.cu) live in VMM memory bound to one multicast object shared by the N
// ranks.  After the backward, rank r owns the float4 slice
// [r n4 / N, (r+1) n4 / N) of the parameter set and, per element e,
//     s  = multimem.ld_reduce.add(G[e])           (the switch sums the N ranks' G sums)
//     g  = s / B_global;  V = mu V + (-eta) g;  W += V   (k_momentum_update_all's sequence)
//     multimem.st G[e] = g, V[e] = V, W[e] = W      (to every rank)
// so each rank moves (1 + 3) / N of the parameter bytes over NVLink instead of
// the 2 (N-1)/N of a ring allreduce plus a full local update pass, and no rank
// ever reads an element another rank writes (slices are disjoint).  Two
// in-stream barriers (multimem.red on a counter every rank holds, then an
// acquire spin on the local copy) order the G sums before the reduce and the
// broadcast stores before the next forward.
//
// Setup (host): rank 0 creates the multicast object and exports it as a POSIX
// file descriptor; the other ranks import it (the descriptor travels over a
// Unix socket, parallel.py); every rank adds its device, then -- after a host
// barrier -- moves its arena into VMM memory, binds it and maps the multicast
// view.  One rank runs the whole sequence locally.  When a single rank cannot
// create a multicast object (a GPU slice without the NVSwitch fabric: the
// driver answers CUDA_ERROR_INVALID_VALUE although the device reports
// multicast support) the state is "local": the same VMM arena, the same slice
// / update / barrier kernels instantiated with plain loads, stores and atomics
// (MC = false) on the rank's own memory -- the multimem path itself needs a
// fabric-attached multi-GPU box.
#pragma once

#include <cuda.h>

#include <cstring>

#include "common.cuh"

namespace lane_b200 {

// ------------------------------------------------------------------ device
template <bool MC>
__device__ __forceinline__ float4 nvls_ld_reduce4(const float* mc) {
    if constexpr (!MC) return *reinterpret_cast<const float4*>(mc);
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(mc)
                 : "memory");
    return v;
}
template <bool MC>
__device__ __forceinline__ void nvls_st4(float* mc, float4 v) {
    if constexpr (!MC) {
        *reinterpret_cast<float4*>(mc) = v;
        return;
    }
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(mc), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// Fused exchange + update over this rank's slice (float4 indices [beg, end) of
// the three regions; mc_* are the multicast views, W / V the local copies).
template <bool MC>
__global__ void __launch_bounds__(256) k_nvls_update(float* mcW, float* mcG, float* mcV, const float4* __restrict__ W,
                                                     const float4* __restrict__ V, unsigned long long beg,
                                                     unsigned long long end, float invB, float neg_eta, float mu) {
    for (unsigned long long e = beg + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < end;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        float4 g = nvls_ld_reduce4<MC>(mcG + 4 * e);
        float4 v = mu == 0.0f ? make_float4(0.f, 0.f, 0.f, 0.f) : V[e];
        float4 w = W[e];
        float* gp = &g.x;
        float* vp = &v.x;
        float* wp = &w.x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float gi = smul(gp[i], invB);
            gp[i] = gi;
            const float step = smul(neg_eta, gi);
            vp[i] = mu == 0.0f ? step : sadd(smul(mu, vp[i]), step);
            wp[i] = sadd(wp[i], vp[i]);
        }
        nvls_st4<MC>(mcG + 4 * e, g);
        nvls_st4<MC>(mcV + 4 * e, v);
        nvls_st4<MC>(mcW + 4 * e, w);
    }
}

// Cross-GPU barrier in the stream: every rank adds 1 to the counter of every
// rank (multimem.red through the switch, release: this GPU's earlier writes
// -- earlier kernels in the stream -- are ordered before it), then waits until
// its local copy holds world x (its barrier count).  `expect` is a per-rank
// device counter, so the kernel replays correctly inside a CUDA graph.
template <bool MC>
__global__ void k_nvls_barrier(unsigned* mc_flag, unsigned* uc_flag, unsigned* expect, int world, int* error) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
    if constexpr (MC)
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], 1;\n" ::"l"(mc_flag) : "memory");
    else
        asm volatile("red.release.sys.global.add.u32 [%0], 1;\n" ::"l"(mc_flag) : "memory");
    const unsigned target = *expect + (unsigned)world;
    *expect = target;
    unsigned seen;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(seen) : "l"(uc_flag) : "memory");
        if ((int)(seen - target) >= 0) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
        if (t - t0 > 10000000000ull) {  // 10 s: a lost rank is an error, never a hang
            if (error) atomicExch(error, 7);
            __trap();
        }
    }
}

// ------------------------------------------------------------------ host
struct NvlsDriver {
    CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long);
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*memRelease)(CUmemGenericAllocationHandle);
    CUresult (*memReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*memFree)(CUdeviceptr, size_t);
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*memUnmap)(CUdeviceptr, size_t);
    CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*memGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
    CUresult (*exportHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
    CUresult (*importHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
    CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice);
};

inline const NvlsDriver& nvls_driver() {
    static NvlsDriver d = [] {
        NvlsDriver x;
        auto get = [](const char* name, auto& fn) {
            void* p = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p ||
                q != cudaDriverEntryPointSuccess)
                throw Error(LANE_ERR_CUDA, std::string("driver entry point unavailable: ") + name);
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
        };
        get("cuMulticastCreate", x.mcCreate);
        get("cuMulticastAddDevice", x.mcAddDevice);
        get("cuMulticastBindMem", x.mcBindMem);
        get("cuMulticastUnbind", x.mcUnbind);
        get("cuMulticastGetGranularity", x.mcGranularity);
        get("cuMemCreate", x.memCreate);
        get("cuMemRelease", x.memRelease);
        get("cuMemAddressReserve", x.memReserve);
        get("cuMemAddressFree", x.memFree);
        get("cuMemMap", x.memMap);
        get("cuMemUnmap", x.memUnmap);
        get("cuMemSetAccess", x.memSetAccess);
        get("cuMemGetAllocationGranularity", x.memGranularity);
        get("cuMemExportToShareableHandle", x.exportHandle);
        get("cuMemImportFromShareableHandle", x.importHandle);
        get("cuDeviceGetAttribute", x.devAttr);
        return x;
    }();
    return d;
}

#define LANE_CU(call)                                                                       \
    do {                                                                                    \
        CUresult r_ = (call);                                                               \
        if (r_ != CUDA_SUCCESS)                                                             \
            throw ::lane_b200::Error(LANE_ERR_CUDA, std::string(#call) + ": CUresult " +   \
                                                        std::to_string((int)r_));           \
    } while (0)

inline bool nvls_supported(int device) {
    try {
        int v = 0;
        if (nvls_driver().devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, device) != CUDA_SUCCESS) return false;
        return v != 0;
    } catch (const Error&) {
        return false;
    }
}

struct NvlsState {
    int rank = 0, world = 1, device = 0;
    bool attached = false, bound = false;
    bool local = false;  // one rank without a multicast object: mcva == uc, MC = false kernels
    CUmemGenericAllocationHandle mc = 0;    // multicast object
    CUmemGenericAllocationHandle phys = 0;  // this rank's arena (VMM)
    size_t bytes = 0;                       // mapped / bound bytes (granularity multiple)
    CUdeviceptr uc = 0, mcva = 0;           // unicast arena VA, multicast VA
    unsigned* expect = nullptr;             // barrier counter (device, per rank)
};

inline size_t nvls_round(size_t n, size_t g) { return (n + g - 1) / g * g; }

inline CUmulticastObjectProp nvls_prop(int world, size_t bytes) {
    CUmulticastObjectProp p;
    std::memset(&p, 0, sizeof(p));
    p.numDevices = (unsigned)world;
    p.size = bytes;
    p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return p;
}

inline size_t nvls_granularity(int world, size_t bytes) {
    const auto& D = nvls_driver();
    CUmulticastObjectProp p = nvls_prop(world, bytes);
    size_t gm = 0;
    LANE_CU(D.mcGranularity(&gm, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ga = 0;
    LANE_CU(D.memGranularity(&ga, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    return std::max(gm, ga);
}

// rank 0: create the multicast object for `bytes` (rounded) over `world` devices
inline void nvls_create(NvlsState& s, int device, int world, size_t bytes) {
    const auto& D = nvls_driver();
    s.world = world;
    s.device = device;
    s.bytes = nvls_round(bytes, nvls_granularity(world, bytes));
    CUmulticastObjectProp p = nvls_prop(world, s.bytes);
    const CUresult r = D.mcCreate(&s.mc, &p);
    if (r != CUDA_SUCCESS && world == 1) {
        s.mc = 0;
        s.local = true;  // see the header: same kernels with plain memory operations
        return;
    }
    LANE_CU(r);
}

inline int nvls_export_fd(const NvlsState& s) {
    int fd = -1;
    if (s.local) return -1;
    LANE_CU(nvls_driver().exportHandle(&fd, s.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    return fd;
}

// ranks != 0: import rank 0's object (size and world are rank 0's)
inline void nvls_import(NvlsState& s, int device, int world, size_t bytes, int fd) {
    s.world = world;
    s.device = device;
    s.bytes = nvls_round(bytes, nvls_granularity(world, bytes));
    LANE_CU(nvls_driver().importHandle(&s.mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                       CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
}

inline void nvls_add_device(NvlsState& s, int rank) {
    if (!s.local) LANE_CU(nvls_driver().mcAddDevice(s.mc, (CUdevice)s.device));
    s.rank = rank;
    s.attached = true;
}

// Every rank, after all ranks added their devices: a VMM arena of s.bytes,
// bound to the multicast object, unicast- and multicast-mapped.  Returns the
// unicast base (the caller copies the old arena in and rebases its pointers).
inline char* nvls_bind(NvlsState& s) {
    const auto& D = nvls_driver();
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = s.device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    LANE_CU(D.memCreate(&s.phys, s.bytes, &ap, 0));
    if (!s.local) LANE_CU(D.mcBindMem(s.mc, 0, s.phys, 0, s.bytes, 0));
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = s.device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    LANE_CU(D.memReserve(&s.uc, s.bytes, 0, 0, 0));
    LANE_CU(D.memMap(s.uc, s.bytes, 0, s.phys, 0));
    LANE_CU(D.memSetAccess(s.uc, s.bytes, &acc, 1));
    if (s.local) {
        s.mcva = s.uc;
    } else {
        LANE_CU(D.memReserve(&s.mcva, s.bytes, 0, 0, 0));
        LANE_CU(D.memMap(s.mcva, s.bytes, 0, s.mc, 0));
        LANE_CU(D.memSetAccess(s.mcva, s.bytes, &acc, 1));
    }
    LANE_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.expect), sizeof(unsigned)));
    LANE_CUDA(cudaMemset(s.expect, 0, sizeof(unsigned)));
    s.bound = true;
    return reinterpret_cast<char*>(s.uc);
}

inline void nvls_release(NvlsState& s) {
    const auto& D = nvls_driver();
    if (s.mcva && s.mcva != s.uc) {
        D.memUnmap(s.mcva, s.bytes);
        D.memFree(s.mcva, s.bytes);
    }
    if (s.uc) {
        D.memUnmap(s.uc, s.bytes);
        D.memFree(s.uc, s.bytes);
    }
    if (s.bound && !s.local) D.mcUnbind(s.mc, (CUdevice)s.device, 0, s.bytes);
    if (s.phys) D.memRelease(s.phys);
    if (s.mc) D.memRelease(s.mc);
    if (s.expect) cudaFree(s.expect);
    s = NvlsState{};
}

}  // namespace lane_b200
