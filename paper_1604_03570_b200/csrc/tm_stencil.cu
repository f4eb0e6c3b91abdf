// Kernels A/C/D: the 7-point stencil sweeps (heat, red-black Gauss-Seidel,
// residual max-norm) over every tile of every FAB in one launch.
//
// One CTA per tile (tm_block).  The tile's planes, grown by one cell in x
// and y, are staged into a kStages-deep shared-memory ring by TMA
// (cp.async.bulk.tensor.4d, one elected thread, mbarrier transaction
// counts).  Threads own fixed (x, y) cells -- one warp covers 32
// consecutive x cells of a row -- and march in z keeping the z-1 and z
// centre values in registers (register-rolling k-march), so each cell costs
// 5 conflict-free shared loads (x+-1, y+-1 of the centre plane, centre of
// the next plane) and one coalesced 8-B store per lane (256 B per warp).
//
// Heat arithmetic is the reference's flux form, operation for operation and
// FMA-free (compiled.py:32-81):
//   fxm = (u[i]-u[i-1])*dxi0, fxp = (u[i+1]-u[i])*dxi0, (y, z likewise)
//   unew = uold + dtD*(((fxp-fxm)*dxi0 + (fyp-fym)*dxi1) + (fzp-fzm)*dxi2)
// so results are bit-identical to the reference (no tolerance needed).
#include <algorithm>
#include <string>
#include <vector>

#include "tm_common.cuh"

namespace {

constexpr int kStages = 4;
constexpr int OP_HEAT = 0, OP_GSRB = 1, OP_RESID = 2;

struct SweepArgs {
    const tm_block *blocks;
    double *out;        // heat: unew, gsrb: phi (in place)
    const double *rhs;  // gsrb / residual
    tm_layout L;        // layout of the staged field
    tm_layout R;        // rhs layout
    double c0, c1, c2, c3;
    int32_t comp0;
    int32_t color;
    unsigned long long *red_out;
    int32_t box_x, box_y, stage_elems;
};

// First column of the staged plane box.  TMA traps (illegal instruction) when
// the innermost box coordinate is not 16-B aligned, so the box starts at the
// even column at or below x0 - 1 and is wide enough for either parity.
__device__ __forceinline__ int box_x_start(const tm_block &blk) { return (blk.x0 - 1) & ~1; }

// Stage plane p (slot-local z = blk.z0 - 1 + p) of field w = slot*ncomp+comp.
__device__ __forceinline__ void issue_plane(const CUtensorMap *map, double *dst, uint64_t *bar, const tm_block &blk,
                                            int p, int w, uint32_t tx_bytes) {
    using namespace tmk;
    mbar_arrive_expect_tx(bar, tx_bytes);
    tma_load_plane(dst, map, bar, box_x_start(blk), blk.y0 - 1, blk.z0 - 1 + p, w);
}

template <int OP, int NWARP, int SEGS>
__global__ void __launch_bounds__(NWARP * 32) sweep_kernel(const __grid_constant__ CUtensorMap map, SweepArgs a) {
    using namespace tmk;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kStages * a.stage_elems * sizeof(double));

    const tm_block blk = a.blocks[blockIdx.x];
    const int comp = a.comp0 + (int)blockIdx.y;
    const int w = blk.slot * a.L.ncomp + comp;
    const int nplanes = blk.nz + 2;
    const int bx = a.box_x;
    const uint32_t tx_bytes = (uint32_t)(a.box_x * a.box_y * sizeof(double));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (tid == 0) {
        prefetch_tensormap(&map);
#pragma unroll
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        const int first = nplanes < kStages ? nplanes : kStages;
        for (int p = 0; p < first; ++p) {
            issue_plane(&map, stages + p * a.stage_elems, &bars[p], blk, p, w, tx_bytes);
        }
    }

    // cells owned by this thread: segment s = warp + NWARP*q -> row s / nxs, x chunk s % nxs
    const int xsh = blk.x0 - box_x_start(blk);  // 1 or 2: smem column of the tile's first cell
    const int nxs = (blk.nx + 31) >> 5;
    const int nseg = blk.ny * nxs;
    int sidx[SEGS], cx[SEGS], cy[SEGS];
    bool act[SEGS];
#pragma unroll
    for (int q = 0; q < SEGS; ++q) {
        const int s = warp + NWARP * q;
        const int y = s / nxs;
        const int x = (s - y * nxs) * 32 + lane;
        act[q] = (s < nseg) && (x < blk.nx);
        cx[q] = x;
        cy[q] = y;
        sidx[q] = (y + 1) * bx + (x + xsh);
    }

    const Strides st = strides_of(a.L);
    const int64_t obase = (int64_t)blk.slot * st.slot + (int64_t)comp * st.comp + (int64_t)blk.z0 * st.plane +
                          (int64_t)blk.y0 * st.row + blk.x0;
    int64_t rbase = 0;
    Strides rs{};
    if (OP != OP_HEAT) {
        rs = strides_of(a.R);
        rbase = (int64_t)blk.slot * rs.slot + (int64_t)(blk.z0 - a.L.nghost + a.R.nghost) * rs.plane +
                (int64_t)(blk.y0 - a.L.nghost + a.R.nghost) * rs.row + (blk.x0 - a.L.xoff + a.R.xoff);
    }

    double um[SEGS], uc[SEGS];
    mbar_wait(&bars[0], 0);
#pragma unroll
    for (int q = 0; q < SEGS; ++q) um[q] = act[q] ? stages[sidx[q]] : 0.0;
    mbar_wait(&bars[1 % kStages], (1 / kStages) & 1);
#pragma unroll
    for (int q = 0; q < SEGS; ++q) uc[q] = act[q] ? stages[(1 % kStages) * a.stage_elems + sidx[q]] : 0.0;
    __syncthreads();
    if (tid == 0 && kStages < nplanes) {
        issue_plane(&map, stages, &bars[0], blk, kStages, w, tx_bytes);
    }

    double vmax = 0.0;
    for (int kk = 0; kk < blk.nz; ++kk) {
        const int pc = kk + 1, pn = kk + 2;
        const double *sc = stages + (pc % kStages) * a.stage_elems;
        const double *sn = stages + (pn % kStages) * a.stage_elems;
        mbar_wait(&bars[pn % kStages], (pn / kStages) & 1);
#pragma unroll
        for (int q = 0; q < SEGS; ++q) {
            if (!act[q]) continue;
            const int i = sidx[q];
            const double xm = sc[i - 1], xp = sc[i + 1], ym = sc[i - bx], yp = sc[i + bx];
            const double un = sn[i];
            const double u0 = uc[q];
            const int64_t cell = (int64_t)kk * st.plane + (int64_t)cy[q] * st.row + cx[q];
            if (OP == OP_HEAT) {
                const double fxm = rn_mul(rn_sub(u0, xm), a.c0), fxp = rn_mul(rn_sub(xp, u0), a.c0);
                const double fym = rn_mul(rn_sub(u0, ym), a.c1), fyp = rn_mul(rn_sub(yp, u0), a.c1);
                const double fzm = rn_mul(rn_sub(u0, um[q]), a.c2), fzp = rn_mul(rn_sub(un, u0), a.c2);
                double s = rn_add(rn_mul(rn_sub(fxp, fxm), a.c0), rn_mul(rn_sub(fyp, fym), a.c1));
                s = rn_add(s, rn_mul(rn_sub(fzp, fzm), a.c2));
                a.out[obase + cell] = rn_add(u0, rn_mul(a.c3, s));
            } else {
                double s = rn_add(xm, xp);
                s = rn_add(s, ym);
                s = rn_add(s, yp);
                s = rn_add(s, um[q]);
                s = rn_add(s, un);
                const int64_t rcell = (int64_t)kk * rs.plane + (int64_t)cy[q] * rs.row + cx[q];
                if (OP == OP_GSRB) {
                    if (((blk.parity + cx[q] + cy[q] + kk) & 1) == a.color) {
                        const double r = __ldg(a.rhs + rbase + rcell);
                        a.out[obase + cell] = __ddiv_rn(rn_add(s, rn_mul(a.c0, r)), 6.0);
                    }
                } else {
                    const double r = __ldg(a.rhs + rbase + rcell);
                    const double res = rn_add(r, __ddiv_rn(rn_sub(s, rn_mul(6.0, u0)), a.c0));
                    vmax = fmax(vmax, fabs(res));
                }
            }
            um[q] = u0;
            uc[q] = un;
        }
        __syncthreads();
        if (tid == 0 && pc + kStages < nplanes) {
            const int st_i = pc % kStages;
            issue_plane(&map, stages + st_i * a.stage_elems, &bars[st_i], blk, pc + kStages, w, tx_bytes);
        }
    }

    if (OP == OP_RESID) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        double *wmax = stages;  // ring is idle after the final __syncthreads of the march
        if (lane == 0) wmax[warp] = vmax;
        __syncthreads();
        if (tid == 0) {
            double m = wmax[0];
            for (int k = 1; k < NWARP; ++k) m = fmax(m, wmax[k]);
            // non-negative doubles order like their bit patterns
            atomicMax(a.red_out, (unsigned long long)__double_as_longlong(m));
        }
    }
}

// Vectorised heat sweep for tiles whose first column is even and whose width
// is a multiple of CPL (the common case: every chopped box of even size).
// Lane l owns CPL consecutive x cells of RPW rows, so shared and global
// accesses are 16-B (double2) wide, the x flux between two cells of a lane is
// computed once, and the z flux of plane k is carried to plane k+1 in
// registers (fz_minus(k+1) == fz_plus(k) bit for bit).  Per cell: 19 FP64
// ops, ~2.5 shared loads, half a 128-bit store.
template <int CPL, int NWARP, int RPW>
__global__ void __launch_bounds__(NWARP * 32) heat_vec_kernel(const __grid_constant__ CUtensorMap map, SweepArgs a) {
    using namespace tmk;
    static_assert(CPL == 2 || CPL == 4, "CPL");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kStages * a.stage_elems * sizeof(double));

    const tm_block blk = a.blocks[blockIdx.x];
    const int comp = a.comp0 + (int)blockIdx.y;
    const int w = blk.slot * a.L.ncomp + comp;
    const int nplanes = blk.nz + 2;
    const int bx = a.box_x;
    const uint32_t tx_bytes = (uint32_t)(a.box_x * a.box_y * sizeof(double));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (tid == 0) {
        prefetch_tensormap(&map);
#pragma unroll
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        const int first = nplanes < kStages ? nplanes : kStages;
        for (int p = 0; p < first; ++p) issue_plane(&map, stages + p * a.stage_elems, &bars[p], blk, p, w, tx_bytes);
    }

    const double c0 = a.c0, c1 = a.c1, c2 = a.c2, c3 = a.c3;
    const bool lane_on = lane * CPL < blk.nx;
    int ci[RPW];
    bool on[RPW];
    double *optr[RPW];
    const Strides st = strides_of(a.L);
    const int64_t obase = (int64_t)blk.slot * st.slot + (int64_t)comp * st.comp + (int64_t)blk.z0 * st.plane +
                          (int64_t)blk.y0 * st.row + blk.x0 + lane * CPL;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int r = warp * RPW + i;
        on[i] = lane_on && r < blk.ny;
        ci[i] = (r + 1) * bx + lane * CPL + 2;  // box starts at x0 - 2 (x0 even)
        optr[i] = a.out + obase + (int64_t)r * st.row;
    }

    double uc[RPW][CPL], fzm[RPW][CPL];
    mbar_wait(&bars[0], 0);
    mbar_wait(&bars[1 % kStages], (1 / kStages) & 1);
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        if (!on[i]) continue;
#pragma unroll
        for (int j = 0; j < CPL; j += 2) {
            const double2 lo = *reinterpret_cast<const double2 *>(stages + ci[i] + j);
            const double2 hi = *reinterpret_cast<const double2 *>(stages + (1 % kStages) * a.stage_elems + ci[i] + j);
            uc[i][j] = hi.x;
            uc[i][j + 1] = hi.y;
            fzm[i][j] = rn_mul(rn_sub(hi.x, lo.x), c2);
            fzm[i][j + 1] = rn_mul(rn_sub(hi.y, lo.y), c2);
        }
    }
    __syncthreads();
    if (tid == 0 && kStages < nplanes) issue_plane(&map, stages, &bars[0], blk, kStages, w, tx_bytes);

    for (int kk = 0; kk < blk.nz; ++kk) {
        const int pc = kk + 1, pn = kk + 2;
        const double *sc = stages + (pc % kStages) * a.stage_elems;
        const double *sn = stages + (pn % kStages) * a.stage_elems;
        mbar_wait(&bars[pn % kStages], (pn / kStages) & 1);
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            if (!on[i]) continue;
            const double *c = sc + ci[i];
            double ym[CPL], yp[CPL], un[CPL], out[CPL];
#pragma unroll
            for (int j = 0; j < CPL; j += 2) {
                const double2 m2 = *reinterpret_cast<const double2 *>(c - bx + j);
                const double2 p2 = *reinterpret_cast<const double2 *>(c + bx + j);
                const double2 n2 = *reinterpret_cast<const double2 *>(sn + ci[i] + j);
                ym[j] = m2.x, ym[j + 1] = m2.y;
                yp[j] = p2.x, yp[j + 1] = p2.y;
                un[j] = n2.x, un[j + 1] = n2.y;
            }
            double fx[CPL + 1];
            fx[0] = rn_mul(rn_sub(uc[i][0], c[-1]), c0);
#pragma unroll
            for (int j = 1; j < CPL; ++j) fx[j] = rn_mul(rn_sub(uc[i][j], uc[i][j - 1]), c0);
            fx[CPL] = rn_mul(rn_sub(c[CPL], uc[i][CPL - 1]), c0);
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
                const double u0 = uc[i][j];
                const double fym = rn_mul(rn_sub(u0, ym[j]), c1), fyp = rn_mul(rn_sub(yp[j], u0), c1);
                const double fzp = rn_mul(rn_sub(un[j], u0), c2);
                double s = rn_add(rn_mul(rn_sub(fx[j + 1], fx[j]), c0), rn_mul(rn_sub(fyp, fym), c1));
                s = rn_add(s, rn_mul(rn_sub(fzp, fzm[i][j]), c2));
                out[j] = rn_add(u0, rn_mul(c3, s));
                fzm[i][j] = fzp;
                uc[i][j] = un[j];
            }
#pragma unroll
            for (int j = 0; j < CPL; j += 2)
                *reinterpret_cast<double2 *>(optr[i] + j) = make_double2(out[j], out[j + 1]);
            optr[i] += st.plane;
        }
        __syncthreads();
        if (tid == 0 && pc + kStages < nplanes) {
            const int st_i = pc % kStages;
            issue_plane(&map, stages + st_i * a.stage_elems, &bars[st_i], blk, pc + kStages, w, tx_bytes);
        }
    }
}

struct KernelCfg {
    int nwarp, segs;
};
constexpr KernelCfg kCfgs[] = {{4, 2}, {8, 2}, {8, 4}, {16, 4}};
constexpr int kMaxSegs = 64;

template <int OP, int NWARP, int SEGS>
int launch_one(const CUtensorMap &map, const SweepArgs &a, int64_t nblocks, int ncomp_grid, size_t smem,
               cudaStream_t s) {
    auto kern = sweep_kernel<OP, NWARP, SEGS>;
    static bool configured = false;  // per instantiation
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute");
        configured = true;
    }
    dim3 grid((unsigned)nblocks, (unsigned)ncomp_grid);
    kern<<<grid, NWARP * 32, smem, s>>>(map, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "sweep launch");
    return TM_OK;
}

template <int CPL, int NWARP, int RPW>
int launch_vec_one(const CUtensorMap &map, const SweepArgs &a, int64_t nblocks, int ncomp_grid, size_t smem,
                   cudaStream_t s) {
    auto kern = heat_vec_kernel<CPL, NWARP, RPW>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute");
        configured = true;
    }
    dim3 grid((unsigned)nblocks, (unsigned)ncomp_grid);
    kern<<<grid, NWARP * 32, smem, s>>>(map, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "heat sweep launch");
    return TM_OK;
}

// vec = 1 + 4*(CPL == 4) + rows config (rows per CTA: 8, 16, 32, 64)
int launch_vec(const CUtensorMap &map, const SweepArgs &a, int vec, int64_t nblocks, int ncomp_grid, size_t smem,
               cudaStream_t s) {
    switch (vec) {
        case 1: return launch_vec_one<2, 4, 2>(map, a, nblocks, ncomp_grid, smem, s);
        case 2: return launch_vec_one<2, 8, 2>(map, a, nblocks, ncomp_grid, smem, s);
        case 3: return launch_vec_one<2, 8, 4>(map, a, nblocks, ncomp_grid, smem, s);
        case 4: return launch_vec_one<2, 16, 4>(map, a, nblocks, ncomp_grid, smem, s);
        case 5: return launch_vec_one<4, 4, 2>(map, a, nblocks, ncomp_grid, smem, s);
        case 6: return launch_vec_one<4, 8, 2>(map, a, nblocks, ncomp_grid, smem, s);
        case 7: return launch_vec_one<4, 8, 4>(map, a, nblocks, ncomp_grid, smem, s);
        default: return launch_vec_one<4, 16, 4>(map, a, nblocks, ncomp_grid, smem, s);
    }
}

template <int OP>
int launch(const CUtensorMap &map, const SweepArgs &a, int cfg, int64_t nblocks, int ncomp_grid, size_t smem,
           cudaStream_t s) {
    switch (cfg) {
        case 0: return launch_one<OP, 4, 2>(map, a, nblocks, ncomp_grid, smem, s);
        case 1: return launch_one<OP, 8, 2>(map, a, nblocks, ncomp_grid, smem, s);
        case 2: return launch_one<OP, 8, 4>(map, a, nblocks, ncomp_grid, smem, s);
        default: return launch_one<OP, 16, 4>(map, a, nblocks, ncomp_grid, smem, s);
    }
}

}  // namespace

struct tm_sweep_plan {
    int64_t nblocks = 0;
    tm_block *d_blocks = nullptr;
    int max_nx = 0, max_ny = 0, max_seg = 0, cfg = 0;
    int vec = 0;  // vectorised heat kernel config, 0 = scalar kernel
    int64_t max_cells = 0;  // largest block
    // small cache of encoded tensor maps keyed by (base pointer, layout)
    struct MapEntry {
        const double *base;
        tm_layout L;
        CUtensorMap map;
    };
    std::vector<MapEntry> maps;
};

namespace {

bool same_layout(const tm_layout &a, const tm_layout &b) {
    return a.nslots == b.nslots && a.ncomp == b.ncomp && a.nghost == b.nghost && a.pitch == b.pitch &&
           a.ny == b.ny && a.nz == b.nz && a.xoff == b.xoff;
}

int plane_map(tm_sweep_plan *p, const tm_layout &L, const double *base, int bx, int by, const CUtensorMap **out) {
    for (auto &m : p->maps)
        if (m.base == base && same_layout(m.L, L)) {
            *out = &m.map;
            return TM_OK;
        }
    if (p->maps.size() >= 8) p->maps.erase(p->maps.begin());
    tm_sweep_plan::MapEntry e;
    e.base = base;
    e.L = L;
    int rc = tmk::encode_plane_map(&e.map, L, base, bx, by);
    if (rc) return rc;
    p->maps.push_back(e);
    *out = &p->maps.back().map;
    return TM_OK;
}

int prepare(tm_sweep_plan *p, const tm_layout *L, const double *base, const char *who, SweepArgs &a,
            const CUtensorMap **map, size_t &smem) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, std::string(who) + ": null plan");
    int rc = check_layout(L, who);
    if (rc) return rc;
    if (L->nghost < 1) return fail(TM_ERR_INVALID, std::string(who) + ": stencil requires nghost >= 1");
    if (!base) return fail(TM_ERR_INVALID, std::string(who) + ": null field");
    // reductions accept any block; stencil sweeps need blocks that fit a CTA tile
    if (p->max_nx + 4 > 256 || p->max_ny + 2 > 256 || p->max_seg > kMaxSegs)
        return fail(TM_ERR_INVALID, std::string(who) + ": block exceeds the CTA tile limit (split it)");
    const int bx = (p->max_nx + 3 + 1) & ~1;  // x0-2 .. x0+nx: covers both start parities
    const int by = p->max_ny + 2;
    rc = plane_map(p, *L, base, bx, by, map);
    if (rc) return rc;
    a.blocks = p->d_blocks;
    a.L = *L;
    a.box_x = bx;
    a.box_y = by;
    a.stage_elems = ((bx * by + 15) / 16) * 16;
    smem = (size_t)kStages * a.stage_elems * sizeof(double) + kStages * sizeof(uint64_t);
    if (smem > 200 * 1024) return fail(TM_ERR_INVALID, std::string(who) + ": tile plane too large for smem");
    return TM_OK;
}

}  // namespace

extern "C" {

int tm_sweep_plan_create(const tm_block *blocks, int64_t nblocks, tm_sweep_plan **out) {
    using namespace tmk;
    if (!out) return fail(TM_ERR_INVALID, "tm_sweep_plan_create: null out");
    *out = nullptr;
    if (nblocks < 0 || (nblocks > 0 && !blocks)) return fail(TM_ERR_INVALID, "tm_sweep_plan_create: bad arguments");
    if (nblocks > (int64_t)INT32_MAX) return fail(TM_ERR_INVALID, "tm_sweep_plan_create: too many blocks");
    int mx = 1, my = 1, maxseg = 1;
    int64_t maxcells = 0;
    bool even2 = true, even4 = true;
    for (int64_t b = 0; b < nblocks; ++b) {
        const tm_block &k = blocks[b];
        if (k.nx < 1 || k.ny < 1 || k.nz < 1 || k.slot < 0 || k.x0 < 0 || k.y0 < 0 || k.z0 < 0)
            return fail(TM_ERR_INVALID, "tm_sweep_plan_create: malformed block " + std::to_string(b));
        mx = std::max(mx, k.nx);
        my = std::max(my, k.ny);
        maxcells = std::max(maxcells, (int64_t)k.nx * k.ny * k.nz);
        maxseg = std::max(maxseg, k.ny * ((k.nx + 31) / 32));
        even2 = even2 && (k.x0 % 2 == 0) && (k.nx % 2 == 0);
        even4 = even4 && (k.x0 % 2 == 0) && (k.nx % 4 == 0);
    }
    tm_sweep_plan *p = new tm_sweep_plan();
    p->nblocks = nblocks;
    p->max_nx = mx;
    p->max_ny = my;
    p->max_seg = maxseg;
    p->max_cells = maxcells;
    const int rows_cfg = my <= 8 ? 0 : my <= 16 ? 1 : my <= 32 ? 2 : my <= 64 ? 3 : -1;
    if (rows_cfg >= 0 && even2 && mx <= 64) p->vec = 1 + rows_cfg;
    else if (rows_cfg >= 0 && even4 && mx <= 128) p->vec = 5 + rows_cfg;
    p->cfg = 3;
    for (int c = 0; c < 4; ++c)
        if (maxseg <= kCfgs[c].nwarp * kCfgs[c].segs) {
            p->cfg = c;
            break;
        }
    if (nblocks > 0) {
        cudaError_t e = cudaMalloc(&p->d_blocks, sizeof(tm_block) * nblocks);
        if (e == cudaSuccess) e = cudaMemcpy(p->d_blocks, blocks, sizeof(tm_block) * nblocks, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(p->d_blocks);
            delete p;
            return cuda_fail(e, "tm_sweep_plan_create");
        }
    }
    *out = p;
    return TM_OK;
}

int tm_sweep_plan_destroy(tm_sweep_plan *plan) {
    if (!plan) return TM_OK;
    // tables may still be read by queued launches on any stream: drain before freeing
    cudaDeviceSynchronize();
    cudaFree(plan->d_blocks);
    delete plan;
    return TM_OK;
}

int tm_heat_sweep(tm_sweep_plan *plan, const tm_layout *layout, const double *uold, double *unew, int32_t comp0,
                  int32_t ncomp_sweep, double dxi0, double dxi1, double dxi2, double dtD, void *stream) {
    using namespace tmk;
    SweepArgs a{};
    const CUtensorMap *map;
    size_t smem;
    int rc = prepare(plan, layout, uold, "tm_heat_sweep", a, &map, smem);
    if (rc) return rc;
    if (!unew || unew == uold) return fail(TM_ERR_INVALID, "tm_heat_sweep: unew must be a distinct buffer");
    if (comp0 < 0 || ncomp_sweep < 1 || comp0 + ncomp_sweep > layout->ncomp)
        return fail(TM_ERR_INVALID, "tm_heat_sweep: component range out of bounds");
    if (plan->nblocks == 0) return TM_OK;
    a.out = unew;
    a.c0 = dxi0;
    a.c1 = dxi1;
    a.c2 = dxi2;
    a.c3 = dtD;
    a.comp0 = comp0;
    if (plan->vec > 0)
        return launch_vec(*map, a, plan->vec, plan->nblocks, ncomp_sweep, smem, as_stream(stream));
    return launch<OP_HEAT>(*map, a, plan->cfg, plan->nblocks, ncomp_sweep, smem, as_stream(stream));
}

int tm_gsrb_color(tm_sweep_plan *plan, const tm_layout *phi_layout, double *phi, const tm_layout *rhs_layout,
                  const double *rhs, int32_t color, double h2, void *stream) {
    using namespace tmk;
    SweepArgs a{};
    const CUtensorMap *map;
    size_t smem;
    int rc = prepare(plan, phi_layout, phi, "tm_gsrb_color", a, &map, smem);
    if (rc) return rc;
    rc = check_layout(rhs_layout, "tm_gsrb_color(rhs)");
    if (rc) return rc;
    if (!rhs || (color != 0 && color != 1)) return fail(TM_ERR_INVALID, "tm_gsrb_color: bad rhs or color");
    if (plan->nblocks == 0) return TM_OK;
    a.out = phi;
    a.rhs = rhs;
    a.R = *rhs_layout;
    a.c0 = h2;
    a.color = color;
    return launch<OP_GSRB>(*map, a, plan->cfg, plan->nblocks, 1, smem, as_stream(stream));
}

int tm_residual_maxnorm(tm_sweep_plan *plan, const tm_layout *phi_layout, const double *phi,
                        const tm_layout *rhs_layout, const double *rhs, double h2, double *d_out, void *stream) {
    using namespace tmk;
    SweepArgs a{};
    const CUtensorMap *map;
    size_t smem;
    int rc = prepare(plan, phi_layout, phi, "tm_residual_maxnorm", a, &map, smem);
    if (rc) return rc;
    rc = check_layout(rhs_layout, "tm_residual_maxnorm(rhs)");
    if (rc) return rc;
    if (!rhs || !d_out) return fail(TM_ERR_INVALID, "tm_residual_maxnorm: null rhs/out");
    cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(double), as_stream(stream));
    if (e != cudaSuccess) return cuda_fail(e, "tm_residual_maxnorm memset");
    if (plan->nblocks == 0) return TM_OK;
    a.rhs = rhs;
    a.R = *rhs_layout;
    a.c0 = h2;
    a.red_out = reinterpret_cast<unsigned long long *>(d_out);
    return launch<OP_RESID>(*map, a, plan->cfg, plan->nblocks, 1, smem, as_stream(stream));
}

}  // extern "C"

extern "C" int tm_internal_plan_blocks(const tm_sweep_plan *p, const tm_block **d_blocks, int64_t *n) {
    *d_blocks = p->d_blocks;
    *n = p->nblocks;
    return TM_OK;
}

extern "C" int64_t tm_internal_plan_max_cells(const tm_sweep_plan *p) { return p->max_cells; }
