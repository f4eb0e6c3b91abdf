// Peer-memory plumbing of the NVLink halo path (include/tilemesh_b200.h,
// "peer halos"): CUDA IPC export / import of a rank's field storage, and the
// per-step device-side barrier that orders the ranks' march launches.
//
// The reference is single-process; the seam is fill_boundary's remote ghost
// copies (/root/reference/pkg/src/tilemesh/level.py:297-323), which in the
// peer path become TMA loads of the neighbour rank's valid cells inside the
// march kernel (tm_march.cu, nbr_src / issue_nbr).  What remains between two
// steps is a synchronisation: every peer must have finished the step that
// wrote the field we read next, and finished reading the field we overwrite.
#include <cstring>
#include <string>

#include "tm_common.cuh"

namespace {

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

PFN_getAddressRange address_range() {
    static PFN_getAddressRange fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_getAddressRange>(f);
        return (PFN_getAddressRange) nullptr;
    }();
    return fn;
}

__device__ __forceinline__ void red_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One warp; lane i < npeers serves peer i.  Launched with programmatic stream serialization
// (its launch overlaps the march before it): griddepcontrol.wait returns once that march has
// completed with its writes visible, the system-scope release publishes them to the peers,
// the acquire orders the peers' writes before the kernels after us (the next march waits for
// this grid to complete).
__global__ void peer_barrier_kernel(uint64_t *inbox, uint64_t *const *peer_inbox, const int32_t *peer_ranks,
                                    int32_t npeers, int32_t my_rank, uint64_t *epoch, int32_t *status,
                                    int64_t timeout_ns) {
    __shared__ uint64_t target;
    const int lane = threadIdx.x;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next march's prologue may start
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0) {
        target = *epoch + 1;
        *epoch = target;
    }
    __syncwarp();
    const uint64_t e = target;
    if (lane < npeers) {
        // the release is the only system-scope fence (an extra fence.acq_rel.sys costs ~1.3 us:
        // tools/micro/barrier_probe.cu)
        red_release_sys(peer_inbox[lane] + my_rank, 1ull);
        const uint64_t *mine = inbox + peer_ranks[lane];
        const uint64_t t0 = globaltimer();
        while (ld_acquire_sys(mine) < e) {
            if ((int64_t)(globaltimer() - t0) > timeout_ns) {
                atomicExch(status, 1);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
}

}  // namespace

extern "C" {

int tm_ipc_export(const void *ptr, uint8_t *handle64, int64_t *offset) {
    using namespace tmk;
    if (!ptr || !handle64 || !offset) return fail(TM_ERR_INVALID, "tm_ipc_export: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
    PFN_getAddressRange range = address_range();
    if (!range) return fail(TM_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
    if (r != CUDA_SUCCESS) return fail(TM_ERR_CUDA, "cuMemGetAddressRange failed: " + std::to_string((int)r));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    memcpy(handle64, &h, 64);
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
    return TM_OK;
}

int tm_ipc_open(const uint8_t *handle64, int64_t offset, void **ptr) {
    using namespace tmk;
    if (!handle64 || !ptr || offset < 0) return fail(TM_ERR_INVALID, "tm_ipc_open: bad argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    *ptr = static_cast<char *>(base) + offset;
    return TM_OK;
}

int tm_ipc_close(void *ptr, int64_t offset) {
    using namespace tmk;
    if (!ptr || offset < 0) return fail(TM_ERR_INVALID, "tm_ipc_close: bad argument");
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(ptr) - offset);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
    return TM_OK;
}

int tm_peer_barrier(uint64_t *inbox, uint64_t *const *peer_inbox, const int32_t *peer_ranks, int32_t npeers,
                    int32_t my_rank, uint64_t *epoch, int32_t *status, int64_t timeout_ns, void *stream) {
    using namespace tmk;
    if (npeers < 0 || npeers > TM_MAX_PEERS || my_rank < 0 || my_rank >= TM_MAX_RANKS)
        return fail(TM_ERR_INVALID, "tm_peer_barrier: 0..TM_MAX_PEERS peers, rank < TM_MAX_RANKS");
    if (!inbox || !epoch || !status || (npeers && (!peer_inbox || !peer_ranks)))
        return fail(TM_ERR_INVALID, "tm_peer_barrier: null argument");
    if (timeout_ns <= 0) return fail(TM_ERR_INVALID, "tm_peer_barrier: timeout must be positive");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, peer_barrier_kernel, inbox, peer_inbox, peer_ranks, npeers, my_rank,
                                       epoch, status, timeout_ns);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tm_peer_barrier launch");
    return TM_OK;
}

}  // extern "C"
