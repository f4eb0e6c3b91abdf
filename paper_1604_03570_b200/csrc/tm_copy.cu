// Kernel B: packed tag copies -- one launch moves every FillBoundary tag of a
// MultiFab (reference level.py:290-294 runs one numpy slice copy per tag from
// a Python loop).  The same kernel packs remote-halo tags into a contiguous
// send buffer, unpacks a receive buffer into ghost cells, and scatters /
// gathers domain-shaped arrays: only the addressing of each side (tm_side)
// changes.
//
// Work decomposition: a tag is ey*ez*ncomp rows of ex contiguous cells.  The
// plan cuts every tag into warp tasks of whole rows -- 32 rows per task when
// rows are short (ex <= 16: x-face ghost columns, one row per lane), about
// 512 cells per task when they are long (y/z faces, gathers; lanes across x)
// -- so a row's address is computed once, not per element, and x-face rows,
// which cost a DRAM chunk each whatever their width, are all in flight at
// once.  Warps stride over the task list; the grid is one wave.
#include <algorithm>
#include <string>
#include <vector>

#include "tm_copy_task.cuh"

namespace {

using namespace tmc;

__global__ void __launch_bounds__(kCopyThreads, 3) copy_tags_kernel(double *__restrict__ dst, SideDev ds,
                                                                    const double *__restrict__ src, SideDev ss,
                                                                    const Task *__restrict__ tasks, int64_t ntasks) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * kWarps;
    int64_t k = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    Task nxt;
    if (k < ntasks) nxt = tasks[k];
    for (; k < ntasks; k += nw) {
        const Task tk = nxt;  // the next task's descriptor is in flight while this one copies
        if (k + nw < ntasks) nxt = tasks[k + nw];
        copy_task(tk, dst, ds, src, ss, lane);
    }
}

}  // namespace


// x-face ghost columns (one layer) from a packed x-halo buffer (tm_xh_to_ghosts).  Four
// consecutive threads write the four 16-B pieces of one row's 64-B chunk in the same
// instruction (a warp: 8 whole chunks), so every chunk reaches L2 as one full write.
__global__ void __launch_bounds__(256) xh_ghosts_kernel(double *__restrict__ base, const double *__restrict__ xh,
                                                       int64_t pitch, int64_t plane, int64_t comp_stride,
                                                       int32_t xlo, int32_t xhi, int32_t nyv, int32_t nzv,
                                                       int32_t y0, int32_t z0, int64_t rows) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t4 < 8 * rows; t4 += stride) {
        // t = ((w * nzv + z) * 2 + side) * nyv + y: the xh element order
        const int64_t t = t4 >> 2;
        const int piece = (int)(t4 & 3);
        const int64_t y = t % nyv;
        const int64_t r = t / nyv;
        const int side = (int)(r & 1);
        const int64_t wz = r >> 1;
        const int64_t z = wz % nzv, w = wz / nzv;
        const double v = xh[t];
        double *row = base + w * comp_stride + (z + z0) * plane + (y + y0) * pitch;
        double2 *chunk = reinterpret_cast<double2 *>(row + (side ? xhi : xlo - 8));
        // the ghost is the chunk's first double on the right (x = hi+1), its last on the left
        const bool holds = side ? piece == 0 : piece == 3;
        chunk[piece] = holds ? (side ? make_double2(v, 0.0) : make_double2(0.0, v)) : make_double2(0.0, 0.0);
    }
}

extern "C" {

int tm_copy_plan_create(const tm_copy_tag *tags, int64_t ntags, int32_t ncomp, tm_copy_plan **out) {
    using namespace tmk;
    if (!out) return fail(TM_ERR_INVALID, "tm_copy_plan_create: null out");
    *out = nullptr;
    if (ntags < 0 || ncomp < 1 || (ntags > 0 && !tags))
        return fail(TM_ERR_INVALID, "tm_copy_plan_create: bad arguments");
    if (ntags >= (int64_t)INT32_MAX) return fail(TM_ERR_INVALID, "tm_copy_plan_create: too many tags");
    std::vector<Task> tasks;
    int64_t total = 0;
    for (int64_t t = 0; t < ntags; ++t) {
        const tm_copy_tag &g = tags[t];
        if (g.ex < 1 || g.ey < 1 || g.ez < 1) return fail(TM_ERR_INVALID, "tm_copy_plan_create: empty tag");
        if (ncomp > 65535) return fail(TM_ERR_INVALID, "tm_copy_plan_create: too many components");
        total += (int64_t)g.ex * g.ey * g.ez * ncomp;
        const int64_t per = (uint32_t)g.ex <= kShortRow ? 32 : std::max<int64_t>(1, kLongTaskCells / g.ex);
        for (int32_t c = 0; c < ncomp; ++c)
            for (int32_t z = 0; z < g.ez; ++z)
                for (int32_t y = 0; y < g.ey; y += (int32_t)per)
                    tasks.push_back(Task{g.src_off, g.dst_off, g.ex, g.ey, g.ez, y, z, (uint16_t)c,
                                         (uint16_t)std::min<int64_t>(per, g.ey - y)});
    }
    tm_copy_plan *p = new tm_copy_plan();
    p->ncomp = ncomp;
    p->ntags = ntags;
    p->ntasks = (int64_t)tasks.size();
    p->elements = total;
    if (!tasks.empty()) {
        int dev = 0, nsm = 148, per_sm = 8;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, copy_tags_kernel, kCopyThreads, 0);
        const int64_t want = (p->ntasks + kWarps - 1) / kWarps;
        p->grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * std::max(per_sm, 1)));
        cudaError_t e = cudaMalloc(&p->d_tasks, sizeof(Task) * tasks.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_tasks, tasks.data(), sizeof(Task) * tasks.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(p->d_tasks);
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
    cudaFree(plan->d_tasks);
    delete plan;
    return TM_OK;
}

int64_t tm_copy_plan_elements(const tm_copy_plan *plan) { return plan ? plan->elements : -1; }

int tm_copy_run(const tm_copy_plan *plan, double *dst, const tm_side *dst_side, const double *src,
                const tm_side *src_side, void *stream) {
    using namespace tmk;
    if (!plan || !dst_side || !src_side) return fail(TM_ERR_INVALID, "tm_copy_run: null argument");
    if (plan->ntasks == 0) return TM_OK;
    if (!dst || !src) return fail(TM_ERR_INVALID, "tm_copy_run: null buffer");
    SideDev ds{dst_side->sy, dst_side->sz, dst_side->sc};
    SideDev ss{src_side->sy, src_side->sz, src_side->sc};
    copy_tags_kernel<<<(unsigned)plan->grid, kCopyThreads, 0, as_stream(stream)>>>(dst, ds, src, ss, plan->d_tasks,
                                                                                   plan->ntasks);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tm_copy_run launch");
    return TM_OK;
}

int tm_xh_to_ghosts(const tm_layout *layout, double *base, const double *xh, int32_t nx, void *stream) {
    using namespace tmk;
    int rc = check_layout(layout, "tm_xh_to_ghosts");
    if (rc) return rc;
    const tm_layout &L = *layout;
    if (!base || !xh || nx < 1) return fail(TM_ERR_INVALID, "tm_xh_to_ghosts: bad arguments");
    if (L.nghost != 1)  // the 64-B chunks overwrite the row padding, where deeper ghost layers live
        return fail(TM_ERR_INVALID, "tm_xh_to_ghosts: needs nghost == 1");
    const int32_t xlo = L.xoff, xhi = L.xoff + nx;
    if (xhi % 2 || xhi + 8 > L.pitch || xlo < 8)
        return fail(TM_ERR_INVALID, "tm_xh_to_ghosts: the 64-B ghost chunks must lie inside the row padding");
    const int32_t nyv = L.ny - 2 * L.nghost, nzv = L.nz - 2 * L.nghost;
    const int64_t rows = L.nslots * L.ncomp * (int64_t)nyv * nzv;
    if (rows == 0) return TM_OK;
    const Strides st = strides_of(L);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t blocks = std::min<int64_t>((8 * rows + 255) / 256, (int64_t)sms * 8);
    xh_ghosts_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(base, xh, st.row, st.plane, st.comp, xlo, xhi,
                                                                      nyv, nzv, L.nghost, L.nghost, rows);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "xh_ghosts_kernel launch");
    return TM_OK;
}

}  // extern "C"
