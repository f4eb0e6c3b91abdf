// Kernel W: the 9-point 8th-order Laplacian step ("wide4")
// on the persistent column march.
//
// Reference: kernels.py:218-247 (wide4_step) and compiled.py:102-129
// (wide4_range).  Per cell, with u the old field and s_m(d) = u[-m] + u[+m]
// along direction d (left operand first):
//   sd   = c0*uc + c1*s_1(d) + c2*s_2(d) + c3*s_3(d) + c4*s_4(d)   (left to right)
//   unew = uc + dtD * ((sx*dxi2_0 + sy*dxi2_1) + sz*dxi2_2)
// evaluated with IEEE round-to-nearest multiplies and adds, no FMA
// contraction (-fmad=false, __d*_rn): bit-identical to the reference.
//
// Layout of the work: the march plan's columns (full box width x <= 16 rows x
// full z) split into equal contiguous plane shares per CTA (segments).  A
// producer warp streams plane boxes [x0-4, x0+nx+4) x [y0-4, y0+ny+4) through
// an 8-stage TMA ring; consumer warp r owns row r of the column and lane l the
// cells x = l, l+32, ... (any width up to 128).  The z neighbours come from a
// 9-deep register window per cell (the ±4 planes), so a plane stays in shared
// memory only while it is the centre plane (its x/y neighbours) -- five planes
// are resident at a time, three more are in flight.  Every plane is read from
// DRAM once per column; the x/y halo rows (4 per side) are the only re-reads.
#include <string>

#include "tm_march_plan.cuh"

namespace {

using tmk::Segment;

constexpr int kW4Stages = 8;  // power of two
constexpr int kR = 4;         // stencil radius

struct W4Args {
    const tm_block *cols;
    const Segment *segs;
    const int32_t *seg_begin;
    double *out;
    tm_layout L;
    double c0, c1, c2, c3, c4;
    double d0, d1, d2, dtD;  // 1/dx^2 per direction, D*dt
    int32_t box_x, box_y, stage_elems;
    // SCATTER: face neighbours nbr[slot][-x,+x,-y,+y,-z,+z] (local slot, or < 0: none) and the
    // uniform box extents; cells within 4 of a face are also written into the neighbour's
    // ghost layers of the new field, so the next step needs no FillBoundary
    const int32_t *nbr;
    int32_t nxb, nyb, nzb;
};

// PAIR: lane l owns the adjacent cells 2l, 2l+1 (widths 34..64): the x window of both
// cells is five 16-B shared loads and every y neighbour pair one, instead of a
// scalar load per neighbour per cell.
template <int CPL, int NWARP, bool PAIR = false, bool SCATTER = false>
__global__ void __launch_bounds__((NWARP + 1) * 32, 1)
    wide4_kernel(const __grid_constant__ CUtensorMap map, W4Args a) {
    using namespace tmk;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kW4Stages * a.stage_elems * sizeof(double));
    uint64_t *empty = bars + kW4Stages;

    const int comp = blockIdx.y;
    const int s_begin = a.seg_begin[blockIdx.x], s_end = a.seg_begin[blockIdx.x + 1];
    if (s_begin >= s_end) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bx = a.box_x;
    const uint32_t tx_bytes = (uint32_t)(a.box_x * a.box_y * (int)sizeof(double));

    if (tid == 0) {
        prefetch_tensormap(&map);
#pragma unroll
        for (int s = 0; s < kW4Stages; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&empty[s], NWARP);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NWARP) {  // ---------------- producer warp ----------------
        if (lane == 0) {
            uint32_t p = 0;
            for (int s = s_begin; s < s_end; ++s) {
                const Segment sg = a.segs[s];
                const tm_block c = a.cols[sg.col];
                const int w = c.slot * a.L.ncomp + comp;
                const int n = sg.k1 - sg.k0 + 2 * kR;
                for (int q = 0; q < n; ++q, ++p) {
                    const uint32_t st_i = p & (kW4Stages - 1);
                    if (p >= (uint32_t)kW4Stages) mbar_wait(&empty[st_i], ((p / kW4Stages) - 1) & 1);
                    mbar_arrive_expect_tx(&bars[st_i], tx_bytes);
                    tma_load_plane(stages + st_i * a.stage_elems, &map, &bars[st_i], c.x0 - kR, c.y0 - kR,
                                   c.z0 + sg.k0 - kR + q, w);
                }
            }
        }
        return;
    }

    // ---------------- consumer warps: warp r = row r of the column ----------------
    const uint32_t sbase = smem_u32(stages);
    const uint32_t bfull = smem_u32(bars), bempty = smem_u32(empty);
    const uint32_t sbytes = (uint32_t)a.stage_elems * 8u;
    auto saddr = [&](uint32_t q) { return sbase + (q & (kW4Stages - 1)) * sbytes; };
    auto wait_plane = [&](uint32_t q) { mbar_wait_u32(bfull + (q & (kW4Stages - 1)) * 8u, (q / kW4Stages) & 1u); };
    auto release = [&](uint32_t q) {
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bempty + (q & (kW4Stages - 1)) * 8u);
    };
    const Strides st = strides_of(a.L);
    const double c0 = a.c0, c1 = a.c1, c2 = a.c2, c3 = a.c3, c4 = a.c4;
    const double d0 = a.d0, d1 = a.d1, d2 = a.d2, dtD = a.dtD;
    const int max_ny = a.box_y - 2 * kR;
    const uint32_t ystep = (uint32_t)bx * 8u;
    const uint32_t pstep = (uint32_t)st.plane;  // < 2^31 (host-checked)
    uint32_t g = 0;  // CTA-wide plane counter of the current segment's first plane

    for (int s = s_begin; s < s_end; ++s) {
        const Segment sg = a.segs[s];
        const tm_block c = a.cols[sg.col];
        const int nk = sg.k1 - sg.k0;
        const int r = warp;
        bool on[CPL];
        uint32_t coff[CPL];  // smem byte offset of cell j in a stage (rows past max_ny clamp; never stored)
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
            const int x = PAIR ? min(2 * lane, bx - 2 * kR - 2) + j : lane + 32 * j;
            on[j] = (PAIR ? 2 * lane + j : x) < c.nx && r < c.ny;
            coff[j] = (uint32_t)((min(r, max_ny - 1) + kR) * bx + min(x, bx - 2 * kR - 1) + kR) * 8u;
        }
        double *const orow = a.out + (int64_t)c.slot * st.slot + (int64_t)comp * st.comp + (int64_t)r * st.row;
        uint32_t koff = (uint32_t)((int64_t)(c.z0 + sg.k0) * st.plane + (int64_t)c.y0 * st.row + c.x0 +
                                   (PAIR ? 2 * lane : lane));
        // scatter targets (pointer deltas from the cell's own address), fixed per column
        int64_t dx[CPL], dy = 0, dzl = 0, dzh = 0;
        bool sx_on[CPL], sy_on = false, szl = false, szh = false;
        int zrel = 0;
        if constexpr (SCATTER) {
            const int32_t *nb = a.nbr + 6 * c.slot;
            const int ng = a.L.nghost;
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
                const int xr = c.x0 - a.L.xoff + (PAIR ? 2 * lane + j : lane + 32 * j);
                sx_on[j] = false;
                dx[j] = 0;
                if (xr < kR && nb[0] >= 0) {
                    sx_on[j] = true;
                    dx[j] = (int64_t)(nb[0] - c.slot) * st.slot + a.nxb;
                } else if (xr >= a.nxb - kR && nb[1] >= 0) {
                    sx_on[j] = true;
                    dx[j] = (int64_t)(nb[1] - c.slot) * st.slot - a.nxb;
                }
            }
            const int yr = c.y0 - ng + r;
            if (yr < kR && nb[2] >= 0) {
                sy_on = true;
                dy = (int64_t)(nb[2] - c.slot) * st.slot + (int64_t)a.nyb * st.row;
            } else if (yr >= a.nyb - kR && nb[3] >= 0) {
                sy_on = true;
                dy = (int64_t)(nb[3] - c.slot) * st.slot - (int64_t)a.nyb * st.row;
            }
            szl = nb[4] >= 0;
            szh = nb[5] >= 0;
            dzl = (int64_t)(nb[4] - c.slot) * st.slot + (int64_t)a.nzb * st.plane;
            dzh = (int64_t)(nb[5] - c.slot) * st.slot - (int64_t)a.nzb * st.plane;
            zrel = c.z0 - ng + sg.k0;
        }

        // window w[m] = u at plane k-4+m of this lane's cells; prime with planes k0-4 .. k0+3
        double w[2 * kR + 1][CPL];
#pragma unroll
        for (int q = 0; q < 2 * kR; ++q) {
            wait_plane(g + q);
            const uint32_t sq = saddr(g + q);
#pragma unroll
            for (int j = 0; j < CPL; ++j) w[q][j] = lds_f64(sq + coff[j]);
            if (q < kR || q >= nk + kR) release(g + q);  // halo planes never become a centre
        }
        for (int kk = 0; kk < nk; ++kk) {
            const uint32_t qn = g + (uint32_t)kk + 2 * kR;  // leading edge: plane k+4
            wait_plane(qn);
            {
                const uint32_t sq = saddr(qn);
#pragma unroll
                for (int j = 0; j < CPL; ++j) w[2 * kR][j] = lds_f64(sq + coff[j]);
            }
            if (kk + 2 * kR >= nk + kR) release(qn);  // trailing halo plane: window use only
            const uint32_t sc = saddr(g + (uint32_t)kk + kR);  // centre plane k
            double out[CPL];
            if constexpr (PAIR) {
                const double cm[kR + 1] = {c0, c1, c2, c3, c4};
                const uint32_t p0 = sc + coff[0];  // cell 2l; its x window starts 4 cells left
                double v[2 * kR + 2];
#pragma unroll
                for (int q = 0; q < kR + 1; ++q) lds_f64x2(p0 - 8u * kR + 16u * q, v[2 * q], v[2 * q + 1]);
                double sx[2], sy[2], sz[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const double cu = rn_mul(c0, w[kR][j]);
                    sx[j] = cu;
                    sy[j] = cu;
                    sz[j] = cu;
                }
#pragma unroll
                for (int m = 1; m <= kR; ++m) {
                    double ym0, ym1, yp0, yp1;
                    lds_f64x2(p0 - ystep * m, ym0, ym1);
                    lds_f64x2(p0 + ystep * m, yp0, yp1);
                    sx[0] = rn_add(sx[0], rn_mul(cm[m], rn_add(v[kR - m], v[kR + m])));
                    sx[1] = rn_add(sx[1], rn_mul(cm[m], rn_add(v[kR + 1 - m], v[kR + 1 + m])));
                    sy[0] = rn_add(sy[0], rn_mul(cm[m], rn_add(ym0, yp0)));
                    sy[1] = rn_add(sy[1], rn_mul(cm[m], rn_add(ym1, yp1)));
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        sz[j] = rn_add(sz[j], rn_mul(cm[m], rn_add(w[kR - m][j], w[kR + m][j])));
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const double lap = rn_add(rn_add(rn_mul(sx[j], d0), rn_mul(sy[j], d1)), rn_mul(sz[j], d2));
                    out[j] = rn_add(w[kR][j], rn_mul(dtD, lap));
                }
            } else
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
                const uint32_t p0 = sc + coff[j];
                const double uc = w[kR][j];
                double xm[kR + 1], xp[kR + 1], ym[kR + 1], yp[kR + 1];
#pragma unroll
                for (int m = 1; m <= kR; ++m) {
                    xm[m] = lds_f64(p0 - 8u * m);
                    xp[m] = lds_f64(p0 + 8u * m);
                    ym[m] = lds_f64(p0 - ystep * m);
                    yp[m] = lds_f64(p0 + ystep * m);
                }
                double sx = rn_mul(c0, uc), sy = rn_mul(c0, uc), sz = rn_mul(c0, uc);
                const double cm[kR + 1] = {c0, c1, c2, c3, c4};
#pragma unroll
                for (int m = 1; m <= kR; ++m) {
                    sx = rn_add(sx, rn_mul(cm[m], rn_add(xm[m], xp[m])));
                    sy = rn_add(sy, rn_mul(cm[m], rn_add(ym[m], yp[m])));
                    sz = rn_add(sz, rn_mul(cm[m], rn_add(w[kR - m][j], w[kR + m][j])));
                }
                const double lap = rn_add(rn_add(rn_mul(sx, d0), rn_mul(sy, d1)), rn_mul(sz, d2));
                out[j] = rn_add(uc, rn_mul(dtD, lap));
            }
            release(g + (uint32_t)kk + kR);
            if constexpr (PAIR) {
                if (on[1]) *reinterpret_cast<double2 *>(orow + koff) = make_double2(out[0], out[1]);
            } else {
#pragma unroll
                for (int j = 0; j < CPL; ++j)
                    if (on[j]) orow[koff + 32 * j] = out[j];
            }
            if constexpr (SCATTER) {
                double *const cell = orow + koff;
                const bool zl = szl && zrel < kR, zh = szh && zrel >= a.nzb - kR;
                if constexpr (PAIR) {
                    if (on[1]) {
                        const double2 pr = make_double2(out[0], out[1]);
                        if (sy_on) *reinterpret_cast<double2 *>(cell + dy) = pr;
                        if (zl) *reinterpret_cast<double2 *>(cell + dzl) = pr;
                        if (zh) *reinterpret_cast<double2 *>(cell + dzh) = pr;
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            if (sx_on[j]) cell[j + dx[j]] = out[j];
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < CPL; ++j) {
                        if (!on[j]) continue;
                        double *const cj = cell + 32 * j;
                        if (sy_on) cj[dy] = out[j];
                        if (zl) cj[dzl] = out[j];
                        if (zh) cj[dzh] = out[j];
                        if (sx_on[j]) cj[dx[j]] = out[j];
                    }
                }
                ++zrel;
            }
            koff += pstep;
#pragma unroll
            for (int m = 0; m < 2 * kR; ++m)
#pragma unroll
                for (int j = 0; j < CPL; ++j) w[m][j] = w[m + 1][j];
        }
        g += nk + 2 * kR;
    }
}

template <int CPL, int NWARP, bool PAIR = false, bool SCATTER = false>
int launch_wide4_one(const CUtensorMap &map, const W4Args &a, int nctas, int ncomp, size_t smem, cudaStream_t s) {
    auto kern = wide4_kernel<CPL, NWARP, PAIR, SCATTER>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute(wide4)");
        configured = true;
    }
    kern<<<dim3(nctas, ncomp), (NWARP + 1) * 32, smem, s>>>(map, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "wide4 launch");
    return TM_OK;
}

}  // namespace

namespace {

template <bool SCATTER>
int wide4_dispatch(const CUtensorMap &map, const W4Args &a, const tm_march_plan *p, int ncomp, size_t smem,
                   cudaStream_t s) {
    const int cpl = (p->max_nx + 31) / 32;
    if (cpl == 1) return launch_wide4_one<1, 16, false, SCATTER>(map, a, p->nctas, ncomp, smem, s);
    if (cpl == 2 && p->even) return launch_wide4_one<2, 16, true, SCATTER>(map, a, p->nctas, ncomp, smem, s);
    if (cpl == 2) return launch_wide4_one<2, 16, false, SCATTER>(map, a, p->nctas, ncomp, smem, s);
    if (p->max_ny > 8) return tmk::fail(TM_ERR_INVALID, "tm_wide4_march: columns wider than 64 must be <= 8 rows");
    return launch_wide4_one<4, 8, false, SCATTER>(map, a, p->nctas, ncomp, smem, s);
}

int wide4_common(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew, int32_t ncomp_sweep,
                 const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2, double dtD, const int32_t *d_nbr,
                 const int32_t *box_extents, void *stream, const char *who) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, std::string(who) + ": null plan");
    int rc = check_layout(layout, who);
    if (rc) return rc;
    const tm_layout &L = *layout;
    if (L.nghost < kR || !uold || !unew || uold == unew || !coeffs5)
        return fail(TM_ERR_INVALID,
                    std::string(who) + ": needs nghost >= 4, distinct old/new fields and 5 coefficients");
    if (ncomp_sweep < 1 || ncomp_sweep > L.ncomp) return fail(TM_ERR_INVALID, std::string(who) + ": bad ncomp");
    if (strides_of(L).comp >= ((int64_t)1 << 32))
        return fail(TM_ERR_INVALID, std::string(who) + ": one component of a slot must hold < 2^32 doubles");
    if (d_nbr && (!box_extents || box_extents[0] < 2 * kR || box_extents[1] < 2 * kR || box_extents[2] < 2 * kR))
        return fail(TM_ERR_INVALID, std::string(who) + ": fused halos need uniform boxes of at least 8^3 cells");
    if (p->ncols == 0) return TM_OK;
    if (p->max_nx > 128 || p->max_ny > 16)
        return fail(TM_ERR_INVALID, std::string(who) + ": columns must be <= 128 wide and <= 16 rows");
    W4Args a{};
    a.cols = p->d_cols;
    a.segs = p->d_segs;
    a.seg_begin = p->d_seg_begin;
    a.out = unew;
    a.L = L;
    a.c0 = coeffs5[0];
    a.c1 = coeffs5[1];
    a.c2 = coeffs5[2];
    a.c3 = coeffs5[3];
    a.c4 = coeffs5[4];
    a.d0 = dxi2_0;
    a.d1 = dxi2_1;
    a.d2 = dxi2_2;
    a.dtD = dtD;
    a.box_x = ((p->max_nx + 2 * kR) + 1) & ~1;  // TMA: inner box bytes a multiple of 16
    a.box_y = p->max_ny + 2 * kR;
    a.stage_elems = ((a.box_x * a.box_y + 15) / 16) * 16;
    a.nbr = d_nbr;
    if (d_nbr) {
        a.nxb = box_extents[0];
        a.nyb = box_extents[1];
        a.nzb = box_extents[2];
    }
    // + slack: idle lanes of a partial-width column read (never store) past their row
    const size_t smem = (size_t)kW4Stages * a.stage_elems * sizeof(double) + 2 * kW4Stages * sizeof(uint64_t) + 2048;
    if (smem > 220 * 1024)
        return fail(TM_ERR_INVALID, std::string(who) + ": column plane too large for shared memory");
    CUtensorMap map;
    rc = encode_plane_map(&map, L, uold, a.box_x, a.box_y);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    return d_nbr ? wide4_dispatch<true>(map, a, p, ncomp_sweep, smem, s)
                 : wide4_dispatch<false>(map, a, p, ncomp_sweep, smem, s);
}

}  // namespace

extern "C" {

int tm_wide4_march(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                   int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                   double dtD, void *stream) {
    return wide4_common(p, layout, uold, unew, ncomp_sweep, coeffs5, dxi2_0, dxi2_1, dxi2_2, dtD, nullptr, nullptr,
                        stream, "tm_wide4_march");
}

int tm_wide4_march_fused(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                         int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                         double dtD, const int32_t *d_nbr, const int32_t *box_extents, void *stream) {
    if (!d_nbr) return tmk::fail(TM_ERR_INVALID, "tm_wide4_march_fused: null neighbour table");
    return wide4_common(p, layout, uold, unew, ncomp_sweep, coeffs5, dxi2_0, dxi2_1, dxi2_2, dtD, d_nbr,
                        box_extents, stream, "tm_wide4_march_fused");
}

}  // extern "C"
