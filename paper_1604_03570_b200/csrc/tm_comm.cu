// Inter-GPU halo exchange over NCCL: one communicator per
// process (one process per GPU), and per FillBoundary ONE grouped
// ncclSend / ncclRecv with the neighbour ranks only.
//
// The reference is single-process; its seam is fill_boundary
// (/root/reference/pkg/src/tilemesh/level.py:297-323).  BoxLib's design it
// generalises -- remote ghost data travels in aggregated per-rank buffers --
// is described at /root/reference/PAPER.md:303-314, :549-556.  The packing
// into / unpacking out of those buffers is the copy kernel (tm_copy_run with
// a packed side); this file only moves the packed messages.
//
// NCCL is resolved at run time with dlopen: when PyTorch (or any other user)
// has already loaded libnccl.so.2 the same library is reused
// (RTLD_NOLOAD), so the process never holds two NCCL versions.  The header
// is only used for its types.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tm_common.cuh"

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int *) = nullptr;
    std::string error;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

template <typename F>
bool sym(void *h, const char *name, F &out) {
    out = reinterpret_cast<F>(dlsym(h, name));
    return out != nullptr;
}

const NcclApi *nccl() {
    std::call_once(g_nccl_once, [] {
        void *h = nullptr;
        const char *env = getenv("TM_NCCL_LIB");
        if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            g_nccl.error = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        bool ok = sym(h, "ncclGetUniqueId", g_nccl.GetUniqueId) && sym(h, "ncclCommInitRank", g_nccl.CommInitRank) &&
                  sym(h, "ncclCommDestroy", g_nccl.CommDestroy) && sym(h, "ncclGroupStart", g_nccl.GroupStart) &&
                  sym(h, "ncclGroupEnd", g_nccl.GroupEnd) && sym(h, "ncclSend", g_nccl.Send) &&
                  sym(h, "ncclRecv", g_nccl.Recv) && sym(h, "ncclGetErrorString", g_nccl.GetErrorString) &&
                  sym(h, "ncclGetVersion", g_nccl.GetVersion);
        if (!ok) {
            g_nccl.error = "libnccl.so.2 lacks a required symbol";
            g_nccl.GetUniqueId = nullptr;
        }
    });
    return g_nccl.GetUniqueId ? &g_nccl : nullptr;
}

int nccl_fail(ncclResult_t r, const char *what) {
    const NcclApi *n = nccl();
    return tmk::fail(TM_ERR_CUDA, std::string(what) + ": " + (n ? n->GetErrorString(r) : "nccl unavailable"));
}

}  // namespace

struct tm_comm {
    ncclComm_t comm = nullptr;
    int32_t nranks = 0, rank = 0;
};

struct tm_exchange {
    tm_comm *comm = nullptr;
    std::vector<int32_t> peers;
    std::vector<int64_t> send_off, send_count, recv_off, recv_count;
};

extern "C" {

int tm_comm_nccl_version(int32_t *version) {
    const NcclApi *n = nccl();
    if (!n) return tmk::fail(TM_ERR_CUDA, g_nccl.error);
    if (!version) return tmk::fail(TM_ERR_INVALID, "tm_comm_nccl_version: null out");
    int v = 0;
    ncclResult_t r = n->GetVersion(&v);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetVersion");
    *version = v;
    return TM_OK;
}

int tm_comm_unique_id(uint8_t *out128) {
    const NcclApi *n = nccl();
    if (!n) return tmk::fail(TM_ERR_CUDA, g_nccl.error);
    if (!out128) return tmk::fail(TM_ERR_INVALID, "tm_comm_unique_id: null out");
    ncclUniqueId id;
    ncclResult_t r = n->GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
    return TM_OK;
}

int tm_comm_create(const uint8_t *id128, int32_t nranks, int32_t rank, tm_comm **out) {
    if (!out) return tmk::fail(TM_ERR_INVALID, "tm_comm_create: null out");
    *out = nullptr;
    if (!id128 || nranks < 1 || rank < 0 || rank >= nranks)
        return tmk::fail(TM_ERR_INVALID, "tm_comm_create: bad id / nranks / rank");
    const NcclApi *n = nccl();
    if (!n) return tmk::fail(TM_ERR_CUDA, g_nccl.error);
    ncclUniqueId id;
    memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
    tm_comm *c = new tm_comm();
    ncclResult_t r = n->CommInitRank(&c->comm, nranks, id, rank);  // on the current CUDA device
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return TM_OK;
}

int tm_comm_destroy(tm_comm *c) {
    if (!c) return TM_OK;
    const NcclApi *n = nccl();
    if (n && c->comm) n->CommDestroy(c->comm);
    delete c;
    return TM_OK;
}

int tm_exchange_create(tm_comm *comm, int32_t npeers, const int32_t *peers, const int64_t *send_off,
                       const int64_t *send_count, const int64_t *recv_off, const int64_t *recv_count,
                       tm_exchange **out) {
    if (!out) return tmk::fail(TM_ERR_INVALID, "tm_exchange_create: null out");
    *out = nullptr;
    if (!comm || npeers < 0 || (npeers > 0 && (!peers || !send_off || !send_count || !recv_off || !recv_count)))
        return tmk::fail(TM_ERR_INVALID, "tm_exchange_create: bad arguments");
    tm_exchange *x = new tm_exchange();
    x->comm = comm;
    for (int32_t i = 0; i < npeers; ++i) {
        if (peers[i] < 0 || peers[i] >= comm->nranks || (i > 0 && peers[i] <= peers[i - 1]) || send_off[i] < 0 ||
            send_count[i] < 0 || recv_off[i] < 0 || recv_count[i] < 0) {
            delete x;
            return tmk::fail(TM_ERR_INVALID, "tm_exchange_create: peers must be distinct ascending ranks with "
                                             "non-negative offsets and counts");
        }
        x->peers.push_back(peers[i]);
        x->send_off.push_back(send_off[i]);
        x->send_count.push_back(send_count[i]);
        x->recv_off.push_back(recv_off[i]);
        x->recv_count.push_back(recv_count[i]);
    }
    *out = x;
    return TM_OK;
}

int tm_exchange_destroy(tm_exchange *x) {
    delete x;
    return TM_OK;
}

int tm_halo_exchange(tm_exchange *x, const double *sendbuf, double *recvbuf, void *stream) {
    if (!x) return tmk::fail(TM_ERR_INVALID, "tm_halo_exchange: null exchange");
    const NcclApi *n = nccl();
    if (!n) return tmk::fail(TM_ERR_CUDA, g_nccl.error);
    cudaStream_t s = tmk::as_stream(stream);
    ncclComm_t c = x->comm->comm;
    ncclResult_t r = n->GroupStart();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    ncclResult_t first = ncclSuccess;
    for (size_t i = 0; i < x->peers.size(); ++i) {
        if (x->send_count[i] > 0) {
            r = n->Send(sendbuf + x->send_off[i], (size_t)x->send_count[i], ncclFloat64, x->peers[i], c, s);
            if (r != ncclSuccess && first == ncclSuccess) first = r;
        }
        if (x->recv_count[i] > 0) {
            r = n->Recv(recvbuf + x->recv_off[i], (size_t)x->recv_count[i], ncclFloat64, x->peers[i], c, s);
            if (r != ncclSuccess && first == ncclSuccess) first = r;
        }
    }
    r = n->GroupEnd();
    if (first != ncclSuccess) return nccl_fail(first, "ncclSend/ncclRecv");
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
    return TM_OK;
}

}  // extern "C"
