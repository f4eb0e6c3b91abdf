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

// ---------------------------------------------------------------------------
// Kernel W2: the same step on columns of up to 32 rows (full box width <= 64).
//
// Why: Kernel W's 16-row columns re-read 8 halo rows per 16 (1.5x in y), and its
// fused variant scatters every cell within 4 of a face into the neighbours' ghost
// layers -- 8-B and 32-B partial-sector writes that HBM's ECC turns into
// read-modify-writes (ncu r01: 363 MB read for 273 MB requested).  W2 halves
// the y re-reads (8 per 32 rows) and, in NBR mode, reads every face halo
// straight from the face neighbour's valid cells, so a fused step writes nothing
// but unew's valid cells.
//
// Work: 8 consumer warps; warp w owns rows 4w .. 4w+3 of the column, lane l the
// cell pair (2l, 2l+1) of each row.  The z window (planes k-4 .. k+4 of the
// warp's 8 cells, 144 registers) lives in registers and rotates by renaming (the
// plane loop is unrolled 9x).  A plane's stage stays resident from landing until
// it is the centre plane (its x/y neighbours), then is released; window-only
// planes (the 4 below / above a segment) are released on landing.  A producer
// warpgroup streams the planes (see wide4_col_kernel for the register split).
//
// Stage layout (doubles), bw = stage row width:
//   GHOST (tm_wide4_march, ghosts filled by FillBoundary): one TMA box
//          (nx+8) x (R+8) at (x0-4, y0-4): rows -4 .. R+3, columns -4 .. nx+3.
//   NBR (tm_wide4_march_nbr): rows -4..-1 (4 x nx) | column rows 0..R-1 (R x nx) |
//          rows R..R+3 (4 x nx), then the x halos XL (R x 4) and XH (R x 4), each
//          region 128-B aligned (TMA destination); halo rows/columns/planes come
//          from the face neighbour's valid cells (own ghosts where there is none).
// ---------------------------------------------------------------------------
constexpr int kW2Warps = 8;  // consumer warps (two warpgroups; 16 x 2 rows measured slower: 106 vs 93 us)
constexpr int kW2Rows = 4;   // rows per consumer warp

struct W2Args {
    const tm_block *cols;
    const Segment *segs;
    const int32_t *seg_begin;
    double *out;
    tm_layout L;
    double c0, c1, c2, c3, c4;
    double d0, d1, d2, dtD;
    int32_t bw;                      // stage row width (doubles)
    int32_t stage_elems, off_xl, off_xh;
    uint32_t tx_c, tx_h;             // TMA bytes of a centre plane / a window-only plane
    const int32_t *nbr;              // NBR: face neighbours per slot
    int32_t nxv, nyv, nzv;           // NBR: uniform box extents
    double *gw;                      // GW: uold, whose 4-deep face ghosts the step writes as it loads them
    const int64_t *fcells;           // GW: (dst, src) offsets in uold of the fill's edge/corner cells
    int64_t nfcells;
};

// A CTA's segments as the producer lane needs them, staged in shared memory at kernel
// start (segments past kW2SegCache are read from global memory): dependent global loads
// on the issue path cost ~10 us per C2-shaped step when consumers issued (r02).
constexpr int kW2SegCache = 32;
struct W2Seg {
    int32_t slot, x0, y0, z0, ny, k0, nk, base;  // base: CTA plane counter of the segment's first plane
    int32_t nb[6];                               // face neighbours (NBR)
    int32_t pad[2];
};
static_assert(sizeof(W2Seg) == 64, "W2Seg is four 16-B words");

template <bool NBR>
__device__ __forceinline__ W2Seg w2_seg_global(const W2Args &A, int s, uint32_t base) {
    const tmk::Segment sg = A.segs[s];
    const tm_block c = A.cols[sg.col];
    W2Seg d;
    d.slot = c.slot;
    d.x0 = c.x0;
    d.y0 = c.y0;
    d.z0 = c.z0;
    d.ny = c.ny;
    d.k0 = sg.k0;
    d.nk = sg.k1 - sg.k0;
    d.base = (int32_t)base;
#pragma unroll
    for (int f = 0; f < 6; ++f) d.nb[f] = NBR ? A.nbr[6 * c.slot + f] : -1;
    d.pad[0] = d.pad[1] = 0;
    return d;
}

// Issue CTA plane P of a W2 launch into its stage.  `cur` = the producer's forward cursor
// (segment index relative to the CTA's first, and that segment's first CTA plane).
template <bool NBR>
__device__ __forceinline__ void w2_issue(const W2Args &A, const CUtensorMap *cmap, const CUtensorMap *ymap,
                                         const CUtensorMap *xmap, double *stages, uint64_t *bars,
                                         const W2Seg *cache, int s_begin, int s_end, int32_t *cur, uint32_t P,
                                         int comp) {
    using namespace tmk;
    const int nc = A.L.ncomp, ng = A.L.nghost;
    int i = *cur;
    W2Seg d = i < kW2SegCache ? cache[i] : w2_seg_global<NBR>(A, s_begin + i, 0);
    uint32_t base = i < kW2SegCache ? (uint32_t)d.base : (uint32_t)cur[1];
    while (P >= base + (uint32_t)(d.nk + 2 * kR) && s_begin + i + 1 < s_end) {
        base += (uint32_t)(d.nk + 2 * kR);
        ++i;
        d = i < kW2SegCache ? cache[i] : w2_seg_global<NBR>(A, s_begin + i, base);
    }
    cur[0] = i;
    cur[1] = (int32_t)base;
    const int q = (int)(P - base);
    const int k = d.k0 - kR + q;  // valid plane index
    const int w = d.slot * nc + comp;
    double *stg = stages + (P & (kW4Stages - 1)) * A.stage_elems;
    uint64_t *bar = &bars[P & (kW4Stages - 1)];
    fence_proxy_async_shared();  // generic reads of the stage's last plane before the async overwrite
    if (NBR) {
        int ws = d.slot, zs = d.z0 + k;
        if (k < 0 && d.nb[4] >= 0) {
            ws = d.nb[4];
            zs += A.nzv;
        } else if (k >= A.nzv && d.nb[5] >= 0) {
            ws = d.nb[5];
            zs -= A.nzv;
        }
        const bool centre = q >= kR && q < d.nk + kR;  // always a plane of our own box
        mbar_arrive_expect_tx(bar, centre ? A.tx_c : A.tx_h);
        tma_load_plane(stg + kR * A.bw, cmap, bar, d.x0, d.y0, zs, ws * nc + comp);
        if (centre) {
            if (d.y0 - ng == 0 && d.nb[2] >= 0)
                tma_load_plane(stg, ymap, bar, d.x0, d.y0 - kR + A.nyv, zs, d.nb[2] * nc + comp);
            else
                tma_load_plane(stg, ymap, bar, d.x0, d.y0 - kR, zs, w);
            double *yh = stg + (kR + d.ny) * A.bw;
            if (d.y0 - ng + d.ny == A.nyv && d.nb[3] >= 0)
                tma_load_plane(yh, ymap, bar, d.x0, d.y0 + d.ny - A.nyv, zs, d.nb[3] * nc + comp);
            else
                tma_load_plane(yh, ymap, bar, d.x0, d.y0 + d.ny, zs, w);
            if (d.nb[0] >= 0)
                tma_load_plane(stg + A.off_xl, xmap, bar, d.x0 + A.nxv - kR, d.y0, zs, d.nb[0] * nc + comp);
            else
                tma_load_plane(stg + A.off_xl, xmap, bar, d.x0 - kR, d.y0, zs, w);
            if (d.nb[1] >= 0)
                tma_load_plane(stg + A.off_xh, xmap, bar, d.x0, d.y0, zs, d.nb[1] * nc + comp);
            else
                tma_load_plane(stg + A.off_xh, xmap, bar, d.x0 + A.nxv, d.y0, zs, w);
        }
    } else {
        mbar_arrive_expect_tx(bar, A.tx_c);
        tma_load_plane(stg, cmap, bar, d.x0 - kR, d.y0 - kR, d.z0 + k, w);
    }
}

// GW ghost writer (one warp of the producer warpgroup): walks the CTA's planes in the ring's
// order and, for each stage, copies what the neighbour-halo loads brought in -- the 4 y halo
// rows and the 4 x halo columns of a centre plane, a whole window-only plane beyond the box --
// to the same cells of uold's ghost region, then releases the stage like a consumer.  These
// are exactly the face ghosts a FillBoundary of uold writes (faces whose neighbour is missing
// were loaded from uold's own ghosts and are skipped).  Inlined: it runs after setmaxnreg.dec (40 regs).
__device__ __forceinline__ void w2_ghost_writer(const W2Args &A, const double *stages, uint64_t *bars, uint64_t *empty,
                                             const W2Seg *cache, int s_begin, int s_end, int comp, int lane,
                                             int which) {
    using namespace tmk;
    const Strides st = strides_of(A.L);
    const int ng = A.L.nghost, bw = A.bw;
    int32_t cur[2] = {0, 0};
    int i = 0;
    W2Seg d = cache[0];
    uint32_t base = 0;
    uint32_t total = 0;
    for (int s = s_begin; s < s_end; ++s) total += (uint32_t)(A.segs[s].k1 - A.segs[s].k0 + 2 * kR);
    for (uint32_t P = 0; P < total; ++P) {
        while (P >= base + (uint32_t)(d.nk + 2 * kR)) {
            base += (uint32_t)(d.nk + 2 * kR);
            ++i;
            d = i < kW2SegCache ? cache[i] : w2_seg_global<true>(A, s_begin + i, base);
        }
        (void)cur;
        mbar_wait(&bars[P & (kW4Stages - 1)], (P / kW4Stages) & 1u);
        if ((int)(P & 1) != which) {  // the other writer's plane: release only
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[P & (kW4Stages - 1)]);
            continue;
        }
        const double *stg = stages + (P & (kW4Stages - 1)) * A.stage_elems;
        const int q = (int)(P - base), k = d.k0 - kR + q;  // valid z of the plane
        double *const slot = A.gw + (int64_t)d.slot * st.slot + (int64_t)comp * st.comp + (int64_t)(d.z0 + k) * st.plane;
        const int nx = A.nxv;
        auto rows_out = [&](const double *src, int nrows, int y_first) {  // nrows x nx from a stage region
            if (2 * lane < nx) {  // a row per iteration: lane = cell pair (nx <= 64)
                double2 *dst = reinterpret_cast<double2 *>(slot + (int64_t)y_first * st.row + d.x0) + lane;
                const double2 *sp = reinterpret_cast<const double2 *>(src) + lane;
#pragma unroll 4
                for (int r = 0; r < nrows; ++r) dst[(int64_t)r * (st.row / 2)] = sp[r * (bw / 2)];
            }
        };
        if (q >= kR && q < d.nk + kR) {  // centre plane: y halo rows, x halo columns
            if (d.y0 - ng == 0 && d.nb[2] >= 0) rows_out(stg, kR, d.y0 - kR);
            if (d.y0 - ng + d.ny == A.nyv && d.nb[3] >= 0) rows_out(stg + (kR + d.ny) * bw, kR, d.y0 + d.ny);
            for (int t = lane; t < 2 * d.ny; t += 32) {  // one 32-B run per row and side
                const int side = t / d.ny, r = t - side * d.ny;
                if (d.nb[side] < 0) continue;
                const double *src = stg + (side ? A.off_xh : A.off_xl) + r * kR;
                double *dst = slot + (int64_t)(d.y0 + r) * st.row + (side ? d.x0 + nx : d.x0 - kR);
                reinterpret_cast<double2 *>(dst)[0] = reinterpret_cast<const double2 *>(src)[0];
                reinterpret_cast<double2 *>(dst)[1] = reinterpret_cast<const double2 *>(src)[1];
            }
        } else if ((k < 0 && d.nb[4] >= 0) || (k >= A.nzv && d.nb[5] >= 0)) {  // a ghost plane
            rows_out(stg + kR * bw, d.ny, d.y0);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[P & (kW4Stages - 1)]);
    }
}

// Warp specialisation with register rebalancing: a 9th (producer) warp would put 3 warps on
// one SM sub-partition and cap every thread at 168 registers, but the consumers' window
// alone takes 144.  So the block is three warpgroups: warpgroup 2 is the producer (one
// lane issues every TMA load; setmaxnreg.dec to 40 registers), warpgroups 0-1 are the
// 8 consumer warps (setmaxnreg.inc to 232).  An earlier producer-less variant (the warp
// releasing a stage last issued its refill) put the issue latency on the slowest warp's
// critical path: 95 vs this kernel's time on the fused C2-shaped step (profiles/r02).
template <int V>
struct IC {
    static constexpr int value = V;
};
constexpr int kW2ProdRegs = 40, kW2ConsRegs = 232;

// GW (with NBR): the step is also the preceding FillBoundary of uold.  Every face halo it loads
// from a neighbour is exactly a ghost value of uold: two warps of the producer warpgroup copy
// them from each stage to uold's ghosts (w2_ghost_writer, alternate planes; both release every
// stage), and the fourth copies the fill's edge/corner cells (which the stencil never reads)
// from a flat (dst, src) list of 4-double runs.  (Storing them from the consumers' registers put
// the stores into all nine unrolled plane bodies: 8040 instructions, instruction-cache bound.)
template <bool NBR, bool GW = false>
__global__ void __launch_bounds__((kW2Warps + 4) * 32, 1)
    wide4_col_kernel(const __grid_constant__ CUtensorMap cmap, const __grid_constant__ CUtensorMap ymap,
                     const __grid_constant__ CUtensorMap xmap, W2Args a) {
    using namespace tmk;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // TMA destinations must be 128-B aligned; the static shared arrays below precede the
    // dynamic window, so align explicitly (the launch adds 128 B of slack)
    unsigned char *smem_al = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    double *stages = reinterpret_cast<double *>(smem_al);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_al + (size_t)kW4Stages * a.stage_elems * sizeof(double));
    uint64_t *empty = bars + kW4Stages;
    __shared__ __align__(16) W2Seg seg_cache[kW2SegCache];  // the CTA's first segments

    const int comp = blockIdx.y;
    const int s_begin = a.seg_begin[blockIdx.x], s_end = a.seg_begin[blockIdx.x + 1];
    if (s_begin >= s_end) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (tid == 0) {
        prefetch_tensormap(&cmap);
        if (NBR) {
            prefetch_tensormap(&ymap);
            prefetch_tensormap(&xmap);
        }
#pragma unroll
        for (int s = 0; s < kW4Stages; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&empty[s], kW2Warps + (GW ? 2 : 0));  // GW: the two ghost writers release stages too
        }
        fence_mbar_init();
        uint32_t base = 0;
        for (int i = 0; i < kW2SegCache && s_begin + i < s_end; ++i) {
            seg_cache[i] = w2_seg_global<NBR>(a, s_begin + i, base);
            base += (uint32_t)(seg_cache[i].nk + 2 * kR);
        }
    }
    grid_dep_launch();
    __syncthreads();
    grid_dep_wait();  // previous step complete: its unew is our uold (and vice versa)

    if (warp >= kW2Warps) {  // ---------------- producer warpgroup ----------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kW2ProdRegs));
        if (GW && (warp == kW2Warps + 1 || warp == kW2Warps + 2)) {  // ghost writers (alternate planes)
            w2_ghost_writer(a, stages, bars, empty, seg_cache, s_begin, s_end, comp, lane, warp - kW2Warps - 1);
        } else if (GW && warp == kW2Warps + 3 && blockIdx.y == 0) {  // fill warp (the list covers every component)
            constexpr int kB = 2;  // entries in flight per lane (40 registers in this warpgroup)
            const int64_t stride = (int64_t)gridDim.x * 32;
            for (int64_t i0 = (int64_t)blockIdx.x * 32 + lane; i0 < a.nfcells; i0 += kB * stride) {
                // entries are runs of 4 doubles along x (32-B aligned: 4-deep ghosts, widths % 4)
                longlong2 ds[kB];
                double2 v[kB][2];
#pragma unroll
                for (int b = 0; b < kB; ++b) {
                    const int64_t i = i0 + b * stride;
                    ds[b] = i < a.nfcells ? reinterpret_cast<const longlong2 *>(a.fcells)[i] : make_longlong2(-1, 0);
                }
#pragma unroll
                for (int b = 0; b < kB; ++b)
                    if (ds[b].x >= 0) {
                        v[b][0] = __ldg(reinterpret_cast<const double2 *>(a.gw + ds[b].y));
                        v[b][1] = __ldg(reinterpret_cast<const double2 *>(a.gw + ds[b].y) + 1);
                    }
#pragma unroll
                for (int b = 0; b < kB; ++b)
                    if (ds[b].x >= 0) {
                        reinterpret_cast<double2 *>(a.gw + ds[b].x)[0] = v[b][0];
                        reinterpret_cast<double2 *>(a.gw + ds[b].x)[1] = v[b][1];
                    }
            }
        }
        if (warp == kW2Warps && lane == 0) {
            uint32_t total = 0;
            for (int s = s_begin; s < s_end; ++s) total += (uint32_t)(a.segs[s].k1 - a.segs[s].k0 + 2 * kR);
            int32_t cur[2] = {0, 0};
            for (uint32_t P = 0; P < total; ++P) {
                if (P >= (uint32_t)kW4Stages) mbar_wait(&empty[P & (kW4Stages - 1)], ((P / kW4Stages) - 1) & 1);
                w2_issue<NBR>(a, &cmap, &ymap, &xmap, stages, bars, seg_cache, s_begin, s_end, cur, P, comp);
            }
        }
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kW2ConsRegs));

    // ---------------- consumer warps ----------------
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
    const double c0 = a.c0, d0 = a.d0, d1 = a.d1, d2 = a.d2, dtD = a.dtD;
    const double cm[kR + 1] = {a.c0, a.c1, a.c2, a.c3, a.c4};
    const int RS = a.bw * 8;  // stage row stride in bytes
    const uint32_t pstep = (uint32_t)st.plane;
    const int r0 = warp * kW2Rows;
    uint32_t g = 0;

    for (int s = s_begin; s < s_end; ++s) {
        const Segment sg = a.segs[s];
        const tm_block c = a.cols[sg.col];
        const int nk = sg.k1 - sg.k0;
        const bool wact = r0 < c.ny;  // rows come in groups of 4 (host-checked)
        const int cx = min(2 * lane, c.nx - 2);
        const bool on = wact && 2 * lane < c.nx;
        // byte offsets inside a stage: the warp's first row at this lane's first cell, and the
        // x pairs q = 0..4 (columns cx-4+2q) at that row, with their row strides
        const int rowb = ((r0 + kR) * a.bw + (NBR ? 0 : kR) + cx) * 8;
        int xo[2 * kR / 2 + 1], xs[2 * kR / 2 + 1];
#pragma unroll
        for (int q = 0; q <= kR; ++q) {
            const int cq = cx - kR + 2 * q;
            if (NBR && cq < 0) {
                xo[q] = (a.off_xl + r0 * kR + cq + kR) * 8;
                xs[q] = kR * 8;
            } else if (NBR && cq >= c.nx) {
                xo[q] = (a.off_xh + r0 * kR + cq - c.nx) * 8;
                xs[q] = kR * 8;
            } else {
                xo[q] = rowb + (cq - cx) * 8;
                xs[q] = RS;
            }
        }
        double *const orow =
            a.out + (int64_t)c.slot * st.slot + (int64_t)comp * st.comp + (int64_t)(c.y0 + r0) * st.row + c.x0 + cx;
        uint32_t koff = (uint32_t)((int64_t)(c.z0 + sg.k0) * st.plane);


        double w[2 * kR + 1][kW2Rows][2];  // window slot (q % 9) <- segment plane q
        auto load_rows = [&](uint32_t sb, double (&dst)[kW2Rows][2]) {
#pragma unroll
            for (int i = 0; i < kW2Rows; ++i) lds_f64x2(sb + (uint32_t)(rowb + i * RS), dst[i][0], dst[i][1]);
        };
        // priming: segment planes 0..7 (k0-4 .. k0+3)
#pragma unroll
        for (int q = 0; q < 2 * kR; ++q) {
            wait_plane(g + q);
            if (wact) load_rows(saddr(g + q), w[q]);
            if (q < kR || q >= nk + kR) release(g + q);  // never a centre plane
        }
        auto body = [&](auto rotc, int kk) {
            constexpr int ROT = decltype(rotc)::value;  // kk % 9: window slot of plane q is q % 9
            constexpr int CEN = (ROT + kR) % (2 * kR + 1);
            const uint32_t qn = g + (uint32_t)kk + 2 * kR;  // leading edge: plane k+4
            wait_plane(qn);
            if (wact) load_rows(saddr(qn), w[(ROT + 2 * kR) % (2 * kR + 1)]);
            if (kk + 2 * kR >= nk + kR) release(qn);  // window-only plane
            const uint32_t qc = g + (uint32_t)kk + kR;
            const uint32_t sc = saddr(qc);
            if (wact) {
#pragma unroll
                for (int i = 0; i < kW2Rows; ++i) {
                    double v[2 * kR + 2];  // columns cx-4 .. cx+5 of row i
#pragma unroll
                    for (int q = 0; q <= kR; ++q) {
                        if (q == kR / 2) {
                            v[2 * q] = w[CEN][i][0];
                            v[2 * q + 1] = w[CEN][i][1];
                        } else {
                            lds_f64x2(sc + (uint32_t)(xo[q] + i * xs[q]), v[2 * q], v[2 * q + 1]);
                        }
                    }

                    double sx[2], sy[2], sz[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const double cu = rn_mul(c0, w[CEN][i][j]);
                        sx[j] = cu;
                        sy[j] = cu;
                        sz[j] = cu;
                    }
#pragma unroll
                    for (int m = 1; m <= kR; ++m) {
                        double ym[2], yp[2];
                        if (i - m >= 0) {
                            ym[0] = w[CEN][i - m][0];
                            ym[1] = w[CEN][i - m][1];
                        } else {
                            lds_f64x2(sc + (uint32_t)(rowb + (i - m) * RS), ym[0], ym[1]);
                        }
                        if (i + m < kW2Rows) {
                            yp[0] = w[CEN][i + m][0];
                            yp[1] = w[CEN][i + m][1];
                        } else {
                            lds_f64x2(sc + (uint32_t)(rowb + (i + m) * RS), yp[0], yp[1]);
                        }
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            sx[j] = rn_add(sx[j], rn_mul(cm[m], rn_add(v[kR + j - m], v[kR + j + m])));
                            sy[j] = rn_add(sy[j], rn_mul(cm[m], rn_add(ym[j], yp[j])));
                            sz[j] = rn_add(sz[j], rn_mul(cm[m], rn_add(w[(ROT + kR - m) % (2 * kR + 1)][i][j],
                                                                        w[(ROT + kR + m) % (2 * kR + 1)][i][j])));
                        }
                    }
                    double out[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const double lap = rn_add(rn_add(rn_mul(sx[j], d0), rn_mul(sy[j], d1)), rn_mul(sz[j], d2));
                        out[j] = rn_add(w[CEN][i][j], rn_mul(dtD, lap));
                    }
                    if (on) *reinterpret_cast<double2 *>(orow + (int64_t)i * st.row + koff) = make_double2(out[0], out[1]);
                }
            }
            release(qc);
            koff += pstep;
        };
        // nine bodies per trip: the window slots rotate by renaming, no register moves (a
        // shifted window costs 128 moves per plane: 77.7 vs 70.4 us per fused C2-shaped step)
        {
            int kk = 0;
            for (;;) {
                if (kk >= nk) break;
                body(IC<0>{}, kk++);
                if (kk >= nk) break;
                body(IC<1>{}, kk++);
                if (kk >= nk) break;
                body(IC<2>{}, kk++);
                if (kk >= nk) break;
                body(IC<3>{}, kk++);
                if (kk >= nk) break;
                body(IC<4>{}, kk++);
                if (kk >= nk) break;
                body(IC<5>{}, kk++);
                if (kk >= nk) break;
                body(IC<6>{}, kk++);
                if (kk >= nk) break;
                body(IC<7>{}, kk++);
                if (kk >= nk) break;
                body(IC<8>{}, kk++);
            }
        }
        g += nk + 2 * kR;
    }
}

template <bool NBR, bool GW = false>
int launch_w2(const CUtensorMap &cmap, const CUtensorMap &ymap, const CUtensorMap &xmap, const W2Args &a, int nctas,
              int ncomp, size_t smem, cudaStream_t s) {
    auto kern = wide4_col_kernel<NBR, GW>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute(wide4 W2)");
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nctas, ncomp);
    cfg.blockDim = dim3((kW2Warps + 4) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, cmap, ymap, xmap, a);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "wide4 W2 launch");
    return TM_OK;
}

// Kernel W2 takes plans of columns <= 64 wide (even) whose row counts are multiples of 4, <= 32.
bool w2_eligible(const tm_march_plan *p) {
    return p->even && p->max_nx <= 64 && p->ny_mult4 && p->max_ny <= kW2Warps * kW2Rows;
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

// Kernel W2 launch: GHOST (x/y/z halos from uold's ghost cells) or NBR (from the face
// neighbours' valid cells, d_box = uniform box extents).  `base` carries the coefficients.
template <bool NBR>
int w2_common(const tm_march_plan *p, const tm_layout &L, const double *uold, const W4Args &base, int ncomp_sweep,
              const int32_t *d_box, cudaStream_t s, const int64_t *fill_cells = nullptr, int64_t nfill = -1) {
    using namespace tmk;
    W2Args a{};
    a.cols = p->d_cols;
    a.segs = p->d_segs;
    a.seg_begin = p->d_seg_begin;
    a.out = base.out;
    a.L = L;
    a.c0 = base.c0;
    a.c1 = base.c1;
    a.c2 = base.c2;
    a.c3 = base.c3;
    a.c4 = base.c4;
    a.d0 = base.d0;
    a.d1 = base.d1;
    a.d2 = base.d2;
    a.dtD = base.dtD;
    const int nx = p->max_nx, R = p->max_ny;
    CUtensorMap cmap, ymap, xmap;
    int rc;
    if (NBR) {
        a.bw = nx;
        a.off_xl = ((nx * (R + 2 * kR) + 15) / 16) * 16;
        a.off_xh = a.off_xl + ((kR * R + 15) / 16) * 16;
        a.stage_elems = a.off_xh + ((kR * R + 15) / 16) * 16;
        a.tx_c = (uint32_t)((nx * R + 2 * kR * nx + 2 * kR * R) * 8);
        a.tx_h = (uint32_t)(nx * R * 8);
        a.nbr = base.nbr;
        a.nxv = d_box[0];
        a.nyv = d_box[1];
        a.nzv = d_box[2];
        rc = encode_plane_map(&cmap, L, uold, nx, R);
        if (!rc) rc = encode_plane_map(&ymap, L, uold, nx, kR);
        if (!rc) rc = encode_plane_map(&xmap, L, uold, kR, R);
    } else {
        a.bw = nx + 2 * kR;
        a.stage_elems = ((a.bw * (R + 2 * kR) + 15) / 16) * 16;
        a.tx_c = a.tx_h = (uint32_t)(a.bw * (R + 2 * kR) * 8);
        a.nyv = L.ny - 2 * L.nghost;
        rc = encode_plane_map(&cmap, L, uold, a.bw, R + 2 * kR);
        ymap = xmap = cmap;
    }
    if (rc) return rc;
    // stages + full barriers + release counters + 128 B of alignment slack
    const size_t smem = (size_t)kW4Stages * a.stage_elems * sizeof(double) + 2 * kW4Stages * sizeof(uint64_t) + 128;
    if (smem > 220 * 1024) return fail(TM_ERR_INVALID, "wide4 W2: column plane too large for shared memory");
    if (NBR && nfill >= 0) {  // GW: this step is also uold's FillBoundary
        a.gw = const_cast<double *>(uold);
        a.fcells = fill_cells;
        a.nfcells = nfill;
        return launch_w2<true, true>(cmap, ymap, xmap, a, p->nctas, ncomp_sweep, smem, s);
    }
    return launch_w2<NBR>(cmap, ymap, xmap, a, p->nctas, ncomp_sweep, smem, s);
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
    if (p->max_nx > 128 || p->max_ny > 32)
        return fail(TM_ERR_INVALID, std::string(who) + ": columns must be <= 128 wide and <= 32 rows");
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
    cudaStream_t s = as_stream(stream);
    if (!d_nbr && w2_eligible(p)) return w2_common<false>(p, L, uold, a, ncomp_sweep, nullptr, s);
    if (p->max_ny > 16)
        return fail(TM_ERR_INVALID, std::string(who) + ": columns of more than 16 rows need widths <= 64 and row "
                                                       "counts that are multiples of 4");
    rc = encode_plane_map(&map, L, uold, a.box_x, a.box_y);
    if (rc) return rc;
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

}  // extern "C"

namespace {

int wide4_nbr_impl(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                   int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                   double dtD, const int32_t *d_nbr, const int32_t *box_extents, const int64_t *fill_cells,
                   int64_t nfill, void *stream) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, "tm_wide4_march_nbr: null plan");
    int rc = check_layout(layout, "tm_wide4_march_nbr");
    if (rc) return rc;
    const tm_layout &L = *layout;
    if (L.nghost < kR || !uold || !unew || uold == unew || !coeffs5 || !d_nbr || !box_extents)
        return fail(TM_ERR_INVALID, "tm_wide4_march_nbr: needs nghost >= 4, distinct old/new fields, 5 coefficients, "
                                    "the neighbour table and the box extents");
    if (ncomp_sweep < 1 || ncomp_sweep > L.ncomp) return fail(TM_ERR_INVALID, "tm_wide4_march_nbr: bad ncomp");
    if (strides_of(L).comp >= ((int64_t)1 << 32))
        return fail(TM_ERR_INVALID, "tm_wide4_march_nbr: one component of a slot must hold < 2^32 doubles");
    if (p->ncols == 0) return TM_OK;
    const int nxv = box_extents[0], nyv = box_extents[1], nzv = box_extents[2];
    // full-width columns of one shape, rows in groups of 4, halo boxes landing 128-B aligned
    if (!(w2_eligible(p) && p->uniform_nx && p->uniform_ny && p->x0_common == L.xoff && p->max_nx == nxv &&
          nxv % 4 == 0 && nyv % p->max_ny == 0 && nyv >= kR && nzv >= kR && L.ny - 2 * L.nghost == nyv &&
          L.nz - 2 * L.nghost == nzv))
        return fail(TM_ERR_INVALID, "tm_wide4_march_nbr: needs uniform boxes (width a multiple of 4, <= 64, each "
                                    "extent >= 4) cut into full-width columns of one height (a multiple of 4, <= 32)");
    W4Args a{};
    a.out = unew;
    const double *c = coeffs5;
    a.c0 = c[0];
    a.c1 = c[1];
    a.c2 = c[2];
    a.c3 = c[3];
    a.c4 = c[4];
    a.d0 = dxi2_0;
    a.d1 = dxi2_1;
    a.d2 = dxi2_2;
    a.dtD = dtD;
    a.nbr = d_nbr;
    return w2_common<true>(p, L, uold, a, ncomp_sweep, box_extents, as_stream(stream), fill_cells, nfill);
}

}  // namespace

extern "C" {

int tm_wide4_march_nbr(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                       int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                       double dtD, const int32_t *d_nbr, const int32_t *box_extents, void *stream) {
    return wide4_nbr_impl(p, layout, uold, unew, ncomp_sweep, coeffs5, dxi2_0, dxi2_1, dxi2_2, dtD, d_nbr,
                          box_extents, nullptr, -1, stream);
}

int tm_wide4_march_fill(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                        int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                        double dtD, const int32_t *d_nbr, const int32_t *box_extents, const int64_t *d_fill_cells,
                        int64_t nfill_cells, void *stream) {
    if (!layout || layout->nghost != kR)
        return tmk::fail(TM_ERR_INVALID, "tm_wide4_march_fill: needs exactly 4 ghost layers (it writes all of them)");
    if (nfill_cells < 0 || (nfill_cells > 0 && !d_fill_cells) ||
        (reinterpret_cast<uintptr_t>(d_fill_cells) & 15) != 0)
        return tmk::fail(TM_ERR_INVALID, "tm_wide4_march_fill: bad cell list (16-B aligned int64 pairs)");
    return wide4_nbr_impl(p, layout, uold, unew, ncomp_sweep, coeffs5, dxi2_0, dxi2_1, dxi2_2, dtD, d_nbr,
                          box_extents, d_fill_cells, nfill_cells, stream);
}

int tm_wide4_march_fused(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                         int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                         double dtD, const int32_t *d_nbr, const int32_t *box_extents, void *stream) {
    if (!d_nbr) return tmk::fail(TM_ERR_INVALID, "tm_wide4_march_fused: null neighbour table");
    return wide4_common(p, layout, uold, unew, ncomp_sweep, coeffs5, dxi2_0, dxi2_1, dxi2_2, dtD, d_nbr,
                        box_extents, stream, "tm_wide4_march_fused");
}

}  // extern "C"
