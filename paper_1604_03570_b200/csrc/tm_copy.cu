// Kernel B: packed tag copies -- one launch moves every FillBoundary tag of a
// MultiFab (reference level.py:290-294 runs one numpy slice copy per tag from
// a Python loop).  The same kernel packs remote-halo tags into a contiguous
// send buffer, unpacks a receive buffer into ghost cells, and scatters /
// gathers domain-shaped host arrays: only the addressing of each side
// (tm_side) changes.
//
// Work decomposition: the tag list is cut into work items of ~kItemElems
// elements (cells x components).  An item covers a run of whole small tags
// and/or a slice of one large tag, so a corner tag of 1 cell and a face tag
// of 4096 cells both keep a CTA busy.  Consecutive threads take consecutive
// x cells of a row, so y/z-face rows are coalesced; x-face tags (ex = nghost)
// are strided by the row pitch by nature of the layout.
#include <algorithm>
#include <string>
#include <vector>

#include "tm_common.cuh"

namespace {

constexpr int kCopyThreads = 256;
constexpr int64_t kItemElems = 2048;
constexpr int kBatch = 4;

struct WorkItem {
    int32_t t0, t1;  // first / last tag (inclusive)
    int32_t e0, e1;  // element range inside t0 (from e0) and inside t1 (to e1, exclusive)
};

struct SideDev {
    int64_t sy, sz, sc;
};

__device__ __forceinline__ int64_t side_offset(const SideDev &s, uint32_t x, uint32_t y, uint32_t z, uint32_t c,
                                               uint32_t ex, uint32_t ey, uint32_t ez) {
    if (s.sy == 0) {  // packed per tag
        return (int64_t)x + (int64_t)ex * ((int64_t)y + (int64_t)ey * ((int64_t)z + (int64_t)ez * c));
    }
    return (int64_t)x + s.sy * y + s.sz * z + s.sc * c;
}

__global__ void __launch_bounds__(kCopyThreads) copy_tags_kernel(double *__restrict__ dst, SideDev ds,
                                                                 const double *__restrict__ src, SideDev ss,
                                                                 uint32_t ncomp, const tm_copy_tag *__restrict__ tags,
                                                                 const WorkItem *__restrict__ items) {
    const WorkItem w = items[blockIdx.x];
    for (int32_t t = w.t0; t <= w.t1; ++t) {
        const tm_copy_tag g = tags[t];
        const uint32_t ex = g.ex, ey = g.ey, ez = g.ez;
        const uint32_t E = ex * ey * ez * ncomp;
        const uint32_t b = (t == w.t0) ? (uint32_t)w.e0 : 0u;
        const uint32_t end = (t == w.t1) ? (uint32_t)w.e1 : E;
        for (uint32_t base = b; base < end; base += kCopyThreads * kBatch) {
            double v[kBatch];
            int64_t doff[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const uint32_t e = base + threadIdx.x + u * kCopyThreads;
                doff[u] = -1;
                if (e < end) {
                    const uint32_t x = e % ex;
                    const uint32_t r = e / ex;
                    const uint32_t y = r % ey;
                    const uint32_t r2 = r / ey;
                    const uint32_t z = r2 % ez;
                    const uint32_t c = r2 / ez;
                    v[u] = __ldg(src + g.src_off + side_offset(ss, x, y, z, c, ex, ey, ez));
                    doff[u] = g.dst_off + side_offset(ds, x, y, z, c, ex, ey, ez);
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u)
                if (doff[u] >= 0) dst[doff[u]] = v[u];
        }
    }
}

}  // namespace

struct tm_copy_plan {
    int32_t ncomp = 1;
    int64_t ntags = 0;
    int64_t nitems = 0;
    int64_t elements = 0;
    tm_copy_tag *d_tags = nullptr;
    WorkItem *d_items = nullptr;
};

extern "C" {

int tm_copy_plan_create(const tm_copy_tag *tags, int64_t ntags, int32_t ncomp, tm_copy_plan **out) {
    using namespace tmk;
    if (!out) return fail(TM_ERR_INVALID, "tm_copy_plan_create: null out");
    *out = nullptr;
    if (ntags < 0 || ncomp < 1 || (ntags > 0 && !tags))
        return fail(TM_ERR_INVALID, "tm_copy_plan_create: bad arguments");
    if (ntags >= (int64_t)INT32_MAX) return fail(TM_ERR_INVALID, "tm_copy_plan_create: too many tags");
    std::vector<WorkItem> items;
    int64_t total = 0;
    // greedy cut of the flattened element stream into ~kItemElems pieces
    int64_t acc = 0;
    WorkItem cur{-1, -1, 0, 0};
    for (int64_t t = 0; t < ntags; ++t) {
        const tm_copy_tag &g = tags[t];
        if (g.ex < 1 || g.ey < 1 || g.ez < 1) return fail(TM_ERR_INVALID, "tm_copy_plan_create: empty tag");
        const int64_t E = (int64_t)g.ex * g.ey * g.ez * ncomp;
        if (E >= (int64_t)UINT32_MAX / 2) return fail(TM_ERR_INVALID, "tm_copy_plan_create: tag too large");
        total += E;
        int64_t pos = 0;
        while (pos < E) {
            if (cur.t0 < 0) {
                cur.t0 = (int32_t)t;
                cur.e0 = (int32_t)pos;
                acc = 0;
            }
            const int64_t take = std::min<int64_t>(E - pos, kItemElems - acc);
            pos += take;
            acc += take;
            cur.t1 = (int32_t)t;
            cur.e1 = (int32_t)pos;
            if (acc >= kItemElems) {
                items.push_back(cur);
                cur = WorkItem{-1, -1, 0, 0};
            }
        }
    }
    if (cur.t0 >= 0) items.push_back(cur);
    tm_copy_plan *p = new tm_copy_plan();
    p->ncomp = ncomp;
    p->ntags = ntags;
    p->nitems = (int64_t)items.size();
    p->elements = total;
    if (ntags > 0) {
        cudaError_t e = cudaMalloc(&p->d_tags, sizeof(tm_copy_tag) * ntags);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_items, sizeof(WorkItem) * items.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_tags, tags, sizeof(tm_copy_tag) * ntags, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_items, items.data(), sizeof(WorkItem) * items.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(p->d_tags);
            cudaFree(p->d_items);
            delete p;
            return cuda_fail(e, "tm_copy_plan_create");
        }
    }
    *out = p;
    return TM_OK;
}

int tm_copy_plan_destroy(tm_copy_plan *plan) {
    if (!plan) return TM_OK;
    cudaFree(plan->d_tags);
    cudaFree(plan->d_items);
    delete plan;
    return TM_OK;
}

int64_t tm_copy_plan_elements(const tm_copy_plan *plan) { return plan ? plan->elements : -1; }

int tm_copy_run(const tm_copy_plan *plan, double *dst, const tm_side *dst_side, const double *src,
                const tm_side *src_side, void *stream) {
    using namespace tmk;
    if (!plan || !dst_side || !src_side) return fail(TM_ERR_INVALID, "tm_copy_run: null argument");
    if (plan->nitems == 0) return TM_OK;
    if (!dst || !src) return fail(TM_ERR_INVALID, "tm_copy_run: null buffer");
    SideDev ds{dst_side->sy, dst_side->sz, dst_side->sc};
    SideDev ss{src_side->sy, src_side->sz, src_side->sc};
    copy_tags_kernel<<<(unsigned)plan->nitems, kCopyThreads, 0, as_stream(stream)>>>(
        dst, ds, src, ss, (uint32_t)plan->ncomp, plan->d_tags, plan->d_items);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tm_copy_run launch");
    return TM_OK;
}

}  // extern "C"
