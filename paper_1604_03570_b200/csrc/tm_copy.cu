// Kernel B: packed tag copies -- one launch moves every FillBoundary tag of a
// MultiFab (reference level.py:290-294 runs one numpy slice copy per tag from
// a Python loop).  The same kernel packs remote-halo tags into a contiguous
// send buffer, unpacks a receive buffer into ghost cells, and scatters /
// gathers domain-shaped arrays: only the addressing of each side (tm_side)
// changes.
//
// Work decomposition: all tags' elements (cells x components, x fastest) form
// one flattened stream with a prefix-sum offset per tag.  CTA b owns stream
// elements [b*kItemElems, (b+1)*kItemElems); each thread takes kBatch
// elements strided by the CTA width, locates their tags by binary search in a
// shared-memory copy of the CTA's slice of the prefix array, and issues all
// kBatch loads before any store.  Corner tags of one cell and face tags of
// thousands of cells therefore cost the same per element, and every load of
// a CTA is in flight at once.  Consecutive threads take consecutive x cells,
// so y/z-face rows are coalesced; x-face tags (ex = nghost) are strided by
// the row pitch by nature of the layout.
#include <algorithm>
#include <string>
#include <vector>

#include "tm_common.cuh"

namespace {

constexpr int kCopyThreads = 256;
constexpr int kBatch = 8;
constexpr int64_t kItemElems = (int64_t)kCopyThreads * kBatch;
constexpr int kMaxSpan = 128;  // tags staged in shared memory per CTA

struct WorkItem {
    int32_t t0, t1;  // tags holding the first / last element of the item
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
                                                                 const int64_t *__restrict__ prefix,
                                                                 const WorkItem *__restrict__ items, int64_t total) {
    __shared__ int64_t sp[kMaxSpan + 1];
    __shared__ tm_copy_tag st[kMaxSpan];
    const WorkItem w = items[blockIdx.x];
    const int span = w.t1 - w.t0 + 1;
    const bool staged = span <= kMaxSpan;
    if (staged) {
        for (int i = threadIdx.x; i <= span; i += kCopyThreads) sp[i] = prefix[w.t0 + i];
        for (int i = threadIdx.x; i < span; i += kCopyThreads) st[i] = tags[w.t0 + i];
    }
    __syncthreads();
    const int64_t e0 = (int64_t)blockIdx.x * kItemElems;
    const int64_t e1 = min(e0 + kItemElems, total);
    const int64_t *P = staged ? sp : prefix + w.t0;
    const tm_copy_tag *T = staged ? st : tags + w.t0;

    double v[kBatch];
    int64_t doff[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
        const int64_t e = e0 + threadIdx.x + (int64_t)u * kCopyThreads;
        doff[u] = -1;
        if (e < e1) {
            int lo = 0, hi = span - 1;  // largest i with P[i] <= e
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (P[mid] <= e) lo = mid;
                else hi = mid - 1;
            }
            const tm_copy_tag g = T[lo];
            const uint32_t local = (uint32_t)(e - P[lo]);
            const uint32_t ex = g.ex, ey = g.ey, ez = g.ez;
            const uint32_t x = local % ex;
            const uint32_t r = local / ex;
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

}  // namespace

struct tm_copy_plan {
    int32_t ncomp = 1;
    int64_t ntags = 0;
    int64_t nitems = 0;
    int64_t elements = 0;
    tm_copy_tag *d_tags = nullptr;
    int64_t *d_prefix = nullptr;
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
    std::vector<int64_t> prefix(ntags + 1, 0);
    for (int64_t t = 0; t < ntags; ++t) {
        const tm_copy_tag &g = tags[t];
        if (g.ex < 1 || g.ey < 1 || g.ez < 1) return fail(TM_ERR_INVALID, "tm_copy_plan_create: empty tag");
        const int64_t E = (int64_t)g.ex * g.ey * g.ez * ncomp;
        if (E >= (int64_t)UINT32_MAX) return fail(TM_ERR_INVALID, "tm_copy_plan_create: tag too large");
        prefix[t + 1] = prefix[t] + E;
    }
    const int64_t total = prefix[ntags];
    const int64_t nitems = (total + kItemElems - 1) / kItemElems;
    if (nitems > (int64_t)INT32_MAX) return fail(TM_ERR_INVALID, "tm_copy_plan_create: too many elements");
    std::vector<WorkItem> items(nitems);
    int64_t t = 0;
    for (int64_t b = 0; b < nitems; ++b) {
        const int64_t first = b * kItemElems, last = std::min(total, first + kItemElems) - 1;
        while (prefix[t + 1] <= first) ++t;
        int64_t t1 = t;
        while (prefix[t1 + 1] <= last) ++t1;
        items[b] = WorkItem{(int32_t)t, (int32_t)t1};
    }
    tm_copy_plan *p = new tm_copy_plan();
    p->ncomp = ncomp;
    p->ntags = ntags;
    p->nitems = nitems;
    p->elements = total;
    if (nitems > 0) {
        cudaError_t e = cudaMalloc(&p->d_tags, sizeof(tm_copy_tag) * ntags);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_prefix, sizeof(int64_t) * (ntags + 1));
        if (e == cudaSuccess) e = cudaMalloc(&p->d_items, sizeof(WorkItem) * nitems);
        if (e == cudaSuccess) e = cudaMemcpy(p->d_tags, tags, sizeof(tm_copy_tag) * ntags, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_prefix, prefix.data(), sizeof(int64_t) * (ntags + 1), cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_items, items.data(), sizeof(WorkItem) * nitems, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(p->d_tags);
            cudaFree(p->d_prefix);
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
    // tables may still be read by queued launches on any stream: drain before freeing
    cudaDeviceSynchronize();
    cudaFree(plan->d_tags);
    cudaFree(plan->d_prefix);
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
        dst, ds, src, ss, (uint32_t)plan->ncomp, plan->d_tags, plan->d_prefix, plan->d_items, plan->elements);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tm_copy_run launch");
    return TM_OK;
}

}  // extern "C"
