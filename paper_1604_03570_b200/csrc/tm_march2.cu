// Kernel A3: two forward-Euler heat steps per launch on the column march
// (temporal blocking).
//
// Each CTA marches its columns once and produces u2 = step(step(u0)) for the
// column's cells.  The intermediate field u1 is computed in shared memory on
// the column plus a one-cell ring in x and y (the face neighbours u2 needs),
// one plane ahead of u2; u0 is read two cells deep around the column.  Every
// u1 and u2 value is computed with the reference's flux-form operations in
// the reference order (compiled.py:32-81, FMA-free), so the result is
// bit-identical to two FillBoundary + heat_step rounds: u1 on the ring equals
// what the neighbouring box computes for the same cell from the same inputs.
//
// Per plane step j of a segment: wait for u0 plane k0+j (TMA ring), compute
// u1(k0-1+j) on column + ring (x/y neighbours from the u0 stage, z from the
// carried flux and the next stage) into a 3-slot shared ring, one barrier
// among the consumer warps, then u2(k0-2+j) from the u1 ring (x/y) and
// registers (z).  Consumer warp w owns column row w; lane l owns cells
// l*CPL .. l*CPL+CPL-1; the 2*nx + 2*ny ring cells are spread evenly over the
// warps, at most one per lane, each with its own carried z flux.
//
// Two halo modes:
//   STD    -- u0's two ghost layers are read from storage (the caller fills
//             them, nghost >= 2); only valid cells of u2 are written.
//   STORE  -- fused halo exchange through storage ghosts: as STD, and the
//             epilogue writes the neighbours' ghost cells of the new field
//             (faces two deep, edges one deep), x ghosts as full 64-B chunks.
//   PACKED -- fused halo exchange.  x halos come from a dense buffer
//             xh[w][2*(z+2)+side][y+2][2] (w = slot*ncomp+c, side 0 = x -2,-1,
//             side 1 = x nx, nx+1, y in [-2, ny+1], z in [-2, nz+1]); y/z
//             ghosts from storage.  The epilogue writes every u2 cell within
//             two layers of a box face into the neighbours' halos of the new
//             field -- y/z ghost rows and planes in storage, x halos in the new
//             xh -- faces two deep and edges one deep, which is everything the
//             next launch reads: consecutive launches need no FillBoundary.
#include <string>

#include "tm_march_plan.cuh"

namespace {

using tmk::Segment;

constexpr int kStages2 = 4;  // power of two
constexpr int kU1Slots = 3;

struct March2Args {
    const tm_block *cols;
    const Segment *segs;
    const int32_t *seg_begin;
    double *out;
    tm_layout L;
    double c0, c1, c2, c3;
    int32_t box_x, box_y, stage_elems;  // u0 main plane box and stage stride (doubles)
    int32_t xh_off, xh1_off;            // PACKED: x-halo slices (side 0 / 1) inside a stage: [row][2]
    int32_t u1_x, u1_elems;             // u1 slot: (nx+4) x (ny+2), cell (x, y) at column x+2, row y+1
    const int32_t *nbr27;               // PACKED: neighbour slot per offset (ox,oy,oz), -1 = none
    double *xh_new;                     // PACKED: x halos of the new field
    int32_t nxb, nyb, nzb;              // PACKED: valid extents of every box
};

template <int CPL, int NWARP, int HALO>
__global__ void __launch_bounds__(NWARP * 32, NWARP <= 8 ? 2 : 1)
    march2_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap xmap,
                  March2Args a) {
    using namespace tmk;
    constexpr bool PACKED = HALO == 1;  // x halos from / to the packed buffers
    constexpr bool SCAT = HALO != 0;    // fused halo exchange (scatter into the new field)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    double *u1s = stages + (size_t)kStages2 * a.stage_elems;
    uint64_t *bars = reinterpret_cast<uint64_t *>(u1s + (size_t)kU1Slots * a.u1_elems);

    const int comp = blockIdx.y;
    const int s_begin = a.seg_begin[blockIdx.x], s_end = a.seg_begin[blockIdx.x + 1];
    if (s_begin >= s_end) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bx = a.box_x, by = a.box_y, ux = a.u1_x;
    const uint32_t tx_bytes = (uint32_t)((bx * by + (PACKED ? 4 * by : 0)) * (int)sizeof(double));

    // No producer warp: the per-plane CTA barrier already orders every stage's last
    // read before its refill, so thread 0 issues the TMA loads right after each
    // barrier, up to three planes ahead of the one being consumed.  16 warps with
    // no 17th keep 4 warps per scheduler and 128 registers per thread.
    const int g_ng0 = a.L.nghost;
    int ps = s_begin, pq = 0;  // producer cursor: segment, plane within it
    uint32_t pnext = 0;        // next plane (CTA sequence) to issue
    auto issue_upto = [&](uint32_t last) {
        fence_proxy_async_shared();  // generic-proxy reads of the stages before their async refill
        while (pnext <= last && ps < s_end) {
            const Segment sg = a.segs[ps];
            const tm_block c = a.cols[sg.col];
            const int w = c.slot * a.L.ncomp + comp;
            const uint32_t st_i = pnext & (kStages2 - 1);
            double *stage = stages + st_i * a.stage_elems;
            const int z = c.z0 + sg.k0 - 2 + pq;
            mbar_arrive_expect_tx(&bars[st_i], tx_bytes);
            if (PACKED) {
                tma_load_plane(stage, &map, &bars[st_i], c.x0, c.y0 - 2, z, w);
                // x halos: rows [y0-2, y0+ny+2) of a plane-side are one contiguous run
                const int zh = 2 * (z - g_ng0 + 2), yh = c.y0 - g_ng0;
                tma_load_plane(stage + a.xh_off, &xmap, &bars[st_i], 2 * yh, zh, 0, w);
                tma_load_plane(stage + a.xh1_off, &xmap, &bars[st_i], 2 * yh, zh + 1, 0, w);
            } else {
                tma_load_plane(stage, &map, &bars[st_i], c.x0 - 2, c.y0 - 2, z, w);
            }
            ++pnext;
            if (++pq == sg.k1 - sg.k0 + 4) {
                pq = 0;
                ++ps;
            }
        }
    };
    if (tid == 0) {
        prefetch_tensormap(&map);
        if (PACKED) prefetch_tensormap(&xmap);
#pragma unroll
        for (int s = 0; s < kStages2; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        issue_upto(kStages2 - 1);
    }
    __syncthreads();

    // ---------------- consumer warps ----------------
    const uint32_t sbase = smem_u32(stages), ubase = smem_u32(u1s);
    const uint32_t bfull = smem_u32(bars);
    const uint32_t sbytes = (uint32_t)a.stage_elems * 8u, ubytes = (uint32_t)a.u1_elems * 8u;
    auto saddr = [&](uint32_t q) { return sbase + (q & (kStages2 - 1)) * sbytes; };
    auto wait_plane = [&](uint32_t q) { mbar_wait_u32(bfull + (q & (kStages2 - 1)) * 8u, (q / kStages2) & 1u); };
    const double c0 = a.c0, c1 = a.c1, c2 = a.c2, c3 = a.c3;
    const Strides st = strides_of(a.L);
    const uint32_t ys0 = (uint32_t)bx * 8u, ys1 = (uint32_t)ux * 8u;  // row strides (bytes): u0 main, u1 slot
    const uint32_t pstep = (uint32_t)st.plane;
    const int max_ny = by - 4;
    const int g_ng = a.L.nghost;
    uint32_t g = 0;   // CTA-wide u0 plane counter of the current segment's first plane
    uint32_t gj = 0;  // CTA-wide u1 plane counter (selects the u1 slot across segments)

    // byte offset in a stage of u0 cell (x, y) of a column of width nx
    auto u0at = [&](int x, int y, int nx) -> uint32_t {
        if (!PACKED) return (uint32_t)((y + 2) * bx + x + 2) * 8u;
        if (x < 0) return (uint32_t)(a.xh_off + (y + 2) * 2 + (x + 2)) * 8u;
        if (x >= nx) return (uint32_t)(a.xh1_off + (y + 2) * 2 + (x - nx)) * 8u;
        return (uint32_t)((y + 2) * bx + x) * 8u;
    };
    // one 7-point flux-form update from explicit neighbour offsets within stage sc
    auto point = [&](uint32_t sc, uint32_t oc, uint32_t oxm, uint32_t oxp, uint32_t oym, uint32_t oyp,
                     double below_flux, double above, double &fz_next) -> double {
        const double u = lds_f64(sc + oc);
        const double xm = lds_f64(sc + oxm), xp = lds_f64(sc + oxp);
        const double ym = lds_f64(sc + oym), yp = lds_f64(sc + oyp);
        const double fxm = rn_mul(rn_sub(u, xm), c0), fxp = rn_mul(rn_sub(xp, u), c0);
        const double fym = rn_mul(rn_sub(u, ym), c1), fyp = rn_mul(rn_sub(yp, u), c1);
        const double fzp = rn_mul(rn_sub(above, u), c2);
        double sum = rn_add(rn_mul(rn_sub(fxp, fxm), c0), rn_mul(rn_sub(fyp, fym), c1));
        sum = rn_add(sum, rn_mul(rn_sub(fzp, below_flux), c2));
        fz_next = fzp;
        return rn_add(u, rn_mul(c3, sum));
    };

    for (int s = s_begin; s < s_end; ++s) {
        const Segment sg = a.segs[s];
        const tm_block c = a.cols[sg.col];
        const int nk = sg.k1 - sg.k0;
        const int r = warp;  // column row of this warp
        const int rc = min(r, max_ny - 1);
        const int xi = min(lane * CPL, c.nx - CPL);
        const bool on = lane * CPL < c.nx && r < c.ny;
        // ring cells (the u1 face neighbours of the column): row -1, row ny, column -1,
        // column nx -- spread evenly, at most one per lane, fixed for the whole column
        const int nring = 2 * c.nx + 2 * c.ny;
        const int per_warp = (nring + NWARP - 1) / NWARP;
        const int t = warp * per_warp + lane;
        const bool has_ring = lane < per_warp && t < nring;
        int rx = 0, ry = 0;
        if (has_ring) {
            if (t < c.nx) {
                rx = t;
                ry = -1;
            } else if (t < 2 * c.nx) {
                rx = t - c.nx;
                ry = c.ny;
            } else if (t < 2 * c.nx + c.ny) {
                rx = -1;
                ry = t - 2 * c.nx;
            } else {
                rx = c.nx;
                ry = t - 2 * c.nx - c.ny;
            }
        }
        // u0 stage offsets: main cells (first cell, its x-1, the cell after the last), ring cell
        const uint32_t o0 = u0at(xi, rc, c.nx), o0l = u0at(xi - 1, rc, c.nx), o0r = u0at(xi + CPL, rc, c.nx);
        const uint32_t rcc = u0at(rx, ry, c.nx), rxm = u0at(rx - 1, ry, c.nx), rxp = u0at(rx + 1, ry, c.nx);
        const uint32_t rym = u0at(rx, ry - 1, c.nx), ryp = u0at(rx, ry + 1, c.nx);
        // u1 slot offsets (col = x + 2, row = y + 1)
        const uint32_t o1 = (uint32_t)((rc + 1) * ux + xi + 2) * 8u;
        const uint32_t o1r = (uint32_t)((ry + 1) * ux + rx + 2) * 8u;
        double *const orow = a.out + (int64_t)c.slot * st.slot + (int64_t)comp * st.comp + (int64_t)r * st.row;
        uint32_t koff = (uint32_t)((int64_t)(c.z0 + sg.k0) * st.plane + (int64_t)c.y0 * st.row + c.x0 + xi);
        // PACKED scatter: y layer of this row (per warp), x-halo roles of this lane
        const int32_t *nb = SCAT ? a.nbr27 + 27 * c.slot : nullptr;
        const int yv = c.y0 - g_ng + r;  // valid y of this row
        int oyv = 0, ylay = 3;
        if (SCAT) {
            if (yv < 2) {
                oyv = -1;
                ylay = yv + 1;
            } else if (yv >= a.nyb - 2) {
                oyv = 1;
                ylay = a.nyb - yv;
            }
        }
        const int zv0 = c.z0 - g_ng + sg.k0;  // valid z of the first output plane
        // the y-face target of this row (rows within two layers of a y face), every plane
        bool vyf = false;
        int64_t dyf = 0;
        if (SCAT && oyv != 0) {
            const int T = nb[13 + 3 * oyv];
            vyf = T >= 0;
            dyf = (int64_t)(T - c.slot) * st.slot - (int64_t)oyv * a.nyb * st.row;
        }
        // x halos: the lane holding cells 0,1 (nx-2, nx-1) feeds side 1 (side 0) of the -x (+x)
        // box; pointers for the face target and the (x, y) edge target follow the planes
        const bool x_role = PACKED && a.xh_new && (xi < 2 || xi + CPL > a.nxb - 2) && lane * CPL < c.nx;
        const int xside = xi < 2 ? 1 : 0, xcol0 = xside ? xi : xi - (a.nxb - 2);
        auto xh_ptr = [&](int T, int oy, int oz, int zv) -> double * {
            const int64_t wT = (int64_t)T * a.L.ncomp + comp;
            return a.xh_new + ((wT * 2 * (a.nzb + 4) + 2 * (zv - oz * a.nzb + 2) + xside) * (a.nyb + 4) +
                               (yv - oy * a.nyb + 2)) * 2 + xcol0;
        };
        double *xq0 = nullptr, *xq1 = nullptr;
        if (x_role) {
            const int T0 = nb[xside ? 12 : 14];
            if (T0 >= 0) xq0 = xh_ptr(T0, 0, 0, zv0);
            if (oyv != 0 && ylay == 1) {
                const int T1 = nb[(xside ? 12 : 14) + 3 * oyv];
                if (T1 >= 0) xq1 = xh_ptr(T1, oyv, 0, zv0);
            }
        }
        const int64_t xzstep = 4 * (int64_t)(a.nyb + 4);  // next z of the same side
        // HALO 2 (storage ghosts): x halos as 64-B chunks -- the lanes holding cells [0, 8)
        // write the -x box's columns [nx, nx+8) (ghosts + row padding), those holding
        // [nx-8, nx) the +x box's columns [-8, 0); face rows and (x, y) edge rows
        const bool cl = HALO == 2 && xi < 8 && lane * CPL < c.nx, cr = HALO == 2 && xi + CPL > a.nxb - 8 && lane * CPL < c.nx;
        int64_t dl0 = 0, dl1 = 0, dr0 = 0, dr1 = 0;
        bool vl0 = false, vl1 = false, vr0 = false, vr1 = false;
        if (HALO == 2) {
            const int TL = nb[12], TR = nb[14];
            vl0 = cl && TL >= 0;
            vr0 = cr && TR >= 0;
            dl0 = (int64_t)(TL - c.slot) * st.slot + a.nxb;
            dr0 = (int64_t)(TR - c.slot) * st.slot - a.nxb;
            if (oyv != 0 && ylay == 1) {
                const int TL1 = nb[12 + 3 * oyv], TR1 = nb[14 + 3 * oyv];
                const int64_t dy = -(int64_t)oyv * a.nyb * st.row;
                vl1 = cl && TL1 >= 0;
                vr1 = cr && TR1 >= 0;
                dl1 = (int64_t)(TL1 - c.slot) * st.slot + dy + a.nxb;
                dr1 = (int64_t)(TR1 - c.slot) * st.slot + dy - a.nxb;
            }
        }

        // u0 march state (main cells: centre values + carried z flux; ring cell: carried flux)
        double u0c[CPL], f0[CPL], f0r = 0.0;
        // u1 march state for u2: centre values and carried z flux (main cells)
        double u1c[CPL], f1[CPL];
        {
            wait_plane(g);
            wait_plane(g + 1);
            const uint32_t sA = saddr(g), sB = saddr(g + 1);
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
                u0c[j] = lds_f64(sB + o0 + 8u * j);
                f0[j] = rn_mul(rn_sub(u0c[j], lds_f64(sA + o0 + 8u * j)), c2);
            }
            if (has_ring) f0r = rn_mul(rn_sub(lds_f64(sB + rcc), lds_f64(sA + rcc)), c2);
        }
        for (int j = 0; j < nk + 2; ++j) {
            // ---- u1 at plane k0-1+j: centre stage g+1+j, next stage g+2+j ----
            const uint32_t qc = g + 1 + (uint32_t)j, qn = qc + 1;
            wait_plane(qn);
            const uint32_t sc = saddr(qc), sn = saddr(qn);
            const uint32_t us = ubase + ((gj + (uint32_t)j) % kU1Slots) * ubytes;
            double u1n[CPL], nxt[CPL];
            {
                double ym[CPL], yp[CPL];
                const uint32_t p0 = sc + o0;
#pragma unroll
                for (int jj = 0; jj < CPL; jj += (CPL >= 2 ? 2 : 1)) {
                    if constexpr (CPL >= 2) {
                        lds_f64x2(p0 - ys0 + 8u * jj, ym[jj], ym[jj + 1]);
                        lds_f64x2(p0 + ys0 + 8u * jj, yp[jj], yp[jj + 1]);
                        lds_f64x2(sn + o0 + 8u * jj, nxt[jj], nxt[jj + 1]);
                    } else {
                        ym[jj] = lds_f64(p0 - ys0);
                        yp[jj] = lds_f64(p0 + ys0);
                        nxt[jj] = lds_f64(sn + o0);
                    }
                }
                double fx[CPL + 1];
                fx[0] = rn_mul(rn_sub(u0c[0], lds_f64(sc + o0l)), c0);
#pragma unroll
                for (int jj = 1; jj < CPL; ++jj) fx[jj] = rn_mul(rn_sub(u0c[jj], u0c[jj - 1]), c0);
                fx[CPL] = rn_mul(rn_sub(lds_f64(sc + o0r), u0c[CPL - 1]), c0);
#pragma unroll
                for (int jj = 0; jj < CPL; ++jj) {
                    const double u = u0c[jj];
                    const double fym = rn_mul(rn_sub(u, ym[jj]), c1), fyp = rn_mul(rn_sub(yp[jj], u), c1);
                    const double fzp = rn_mul(rn_sub(nxt[jj], u), c2);
                    double sum = rn_add(rn_mul(rn_sub(fx[jj + 1], fx[jj]), c0), rn_mul(rn_sub(fyp, fym), c1));
                    sum = rn_add(sum, rn_mul(rn_sub(fzp, f0[jj]), c2));
                    u1n[jj] = rn_add(u, rn_mul(c3, sum));
                    f0[jj] = fzp;
                }
            }
            double vr = 0.0;
            if (has_ring) {
                double fz;
                vr = point(sc, rcc, rxm, rxp, rym, ryp, f0r, lds_f64(sn + rcc), fz);
                f0r = fz;
            }
#pragma unroll
            for (int jj = 0; jj < CPL; ++jj) u0c[jj] = nxt[jj];
            // publish u1(k0-1+j); rows >= ny and lanes past nx hold values nobody reads
            if constexpr (CPL >= 2) {
#pragma unroll
                for (int jj = 0; jj < CPL; jj += 2) sts_f64x2(us + o1 + 8u * jj, u1n[jj], u1n[jj + 1]);
            } else {
                sts_f64(us + o1, u1n[0]);
            }
            if (has_ring) sts_f64(us + o1r, vr);
            named_barrier_sync(1, NWARP * 32);
            // every warp is done with planes <= qc: refill up to qn + 3
            if (tid == 0) issue_upto(qn + 3);
            if (j == 0) {
#pragma unroll
                for (int jj = 0; jj < CPL; ++jj) u1c[jj] = u1n[jj];
                continue;
            }
            if (j == 1) {
#pragma unroll
                for (int jj = 0; jj < CPL; ++jj) {
                    f1[jj] = rn_mul(rn_sub(u1n[jj], u1c[jj]), c2);
                    u1c[jj] = u1n[jj];
                }
                continue;
            }
            // ---- u2 at plane k0-2+j from the u1 slot of plane k0-2+j (x/y) and registers (z) ----
            const uint32_t up = ubase + ((gj + (uint32_t)j - 1) % kU1Slots) * ubytes + o1;
            double out[CPL];
            {
                double ym[CPL], yp[CPL];
#pragma unroll
                for (int jj = 0; jj < CPL; jj += (CPL >= 2 ? 2 : 1)) {
                    if constexpr (CPL >= 2) {
                        lds_f64x2(up - ys1 + 8u * jj, ym[jj], ym[jj + 1]);
                        lds_f64x2(up + ys1 + 8u * jj, yp[jj], yp[jj + 1]);
                    } else {
                        ym[jj] = lds_f64(up - ys1);
                        yp[jj] = lds_f64(up + ys1);
                    }
                }
                double fx[CPL + 1];
                fx[0] = rn_mul(rn_sub(u1c[0], lds_f64(up - 8u)), c0);
#pragma unroll
                for (int jj = 1; jj < CPL; ++jj) fx[jj] = rn_mul(rn_sub(u1c[jj], u1c[jj - 1]), c0);
                fx[CPL] = rn_mul(rn_sub(lds_f64(up + 8u * CPL), u1c[CPL - 1]), c0);
#pragma unroll
                for (int jj = 0; jj < CPL; ++jj) {
                    const double u = u1c[jj];
                    const double fym = rn_mul(rn_sub(u, ym[jj]), c1), fyp = rn_mul(rn_sub(yp[jj], u), c1);
                    const double fzp = rn_mul(rn_sub(u1n[jj], u), c2);
                    double sum = rn_add(rn_mul(rn_sub(fx[jj + 1], fx[jj]), c0), rn_mul(rn_sub(fyp, fym), c1));
                    sum = rn_add(sum, rn_mul(rn_sub(fzp, f1[jj]), c2));
                    out[jj] = rn_add(u, rn_mul(c3, sum));
                    f1[jj] = fzp;
                    u1c[jj] = u1n[jj];
                }
            }
            auto put = [&](int64_t delta) {
                if constexpr (CPL >= 2) {
#pragma unroll
                    for (int jj = 0; jj < CPL; jj += 2)
                        *reinterpret_cast<double2 *>(orow + koff + delta + jj) = make_double2(out[jj], out[jj + 1]);
                } else {
                    orow[koff + delta] = out[0];
                }
            };
            if (on) {
                put(0);
                if (SCAT && (HALO == 2 || a.xh_new)) {
                    // every plane: x faces (+ this row's (x, y) edge) and this row's y face
                    auto xput = [&](double *q) {
                        if constexpr (CPL >= 2)
                            *reinterpret_cast<double2 *>(q) = make_double2(out[0], out[1]);
                        else
                            *q = out[0];
                    };
                    if (HALO == 1) {
                        if (xq0) xput(xq0);
                        if (xq1) xput(xq1);
                    } else {
                        if (vl0) put(dl0);
                        if (vr0) put(dr0);
                        if (vl1) put(dl1);
                        if (vr1) put(dr1);
                    }
                    if (vyf) put(dyf);
                    // the two planes next to each z face (warp-uniform, rare): z faces two deep,
                    // (y, z) and (x, z) edges one deep
                    const int zv = zv0 + j - 2;
                    if (zv < 2 || zv >= a.nzb - 2) {
                        const int ozv = zv < 2 ? -1 : 1, zlay = zv < 2 ? zv + 1 : a.nzb - zv;
                        const int64_t dz = -(int64_t)ozv * a.nzb * st.plane;
                        const int Tz = nb[13 + 9 * ozv];
                        if (Tz >= 0) put((int64_t)(Tz - c.slot) * st.slot + dz);
                        if (zlay == 1) {
                            if (oyv != 0 && ylay == 1) {
                                const int Tyz = nb[13 + 3 * oyv + 9 * ozv];
                                if (Tyz >= 0) put((int64_t)(Tyz - c.slot) * st.slot + dz - (int64_t)oyv * a.nyb * st.row);
                            }
                            if (HALO == 1 && x_role) {
                                const int T2 = nb[(xside ? 12 : 14) + 9 * ozv];
                                if (T2 >= 0) xput(xh_ptr(T2, 0, ozv, zv));
                            }
                            if (HALO == 2) {
                                if (cl) {
                                    const int T2 = nb[12 + 9 * ozv];
                                    if (T2 >= 0) put((int64_t)(T2 - c.slot) * st.slot + dz + a.nxb);
                                }
                                if (cr) {
                                    const int T3 = nb[14 + 9 * ozv];
                                    if (T3 >= 0) put((int64_t)(T3 - c.slot) * st.slot + dz - a.nxb);
                                }
                            }
                        }
                    }
                }
            }
            koff += pstep;
            if (xq0) xq0 += xzstep;
            if (xq1) xq1 += xzstep;
        }
        g += (uint32_t)nk + 4;
        gj += (uint32_t)nk + 2;
    }
}

template <int CPL, int NWARP, int HALO>
int launch_march2_one(const CUtensorMap &map, const CUtensorMap &xmap, const March2Args &a, int nctas, int ncomp,
                      size_t smem, cudaStream_t s) {
    auto kern = march2_kernel<CPL, NWARP, HALO>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute(march2)");
        configured = true;
    }
    kern<<<dim3(nctas, ncomp), NWARP * 32, smem, s>>>(map, xmap, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "march2 launch");
    return TM_OK;
}

template <int HALO>
int launch_mode(const CUtensorMap &map, const CUtensorMap &xmap, const March2Args &a, const tm_march_plan *p,
                int ncomp, size_t smem, cudaStream_t s) {
    if (p->max_ny <= 8) {  // 8-row columns: two CTAs per SM
        if (p->max_nx <= 32) return launch_march2_one<1, 8, HALO>(map, xmap, a, p->nctas, ncomp, smem, s);
        return launch_march2_one<2, 8, HALO>(map, xmap, a, p->nctas, ncomp, smem, s);
    }
    if (p->max_nx <= 32) return launch_march2_one<1, 16, HALO>(map, xmap, a, p->nctas, ncomp, smem, s);
    return launch_march2_one<2, 16, HALO>(map, xmap, a, p->nctas, ncomp, smem, s);
}

}  // namespace

extern "C" {

int tm_heat_march2(tm_march_plan *p, const tm_layout *layout, const double *u0, double *u2, int32_t ncomp_sweep,
                   double dxi0, double dxi1, double dxi2, double dtD, const double *xh_old, double *xh_new,
                   const int32_t *d_nbr27, void *stream) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, "tm_heat_march2: null plan");
    int rc = check_layout(layout, "tm_heat_march2");
    if (rc) return rc;
    const tm_layout &L = *layout;
    const bool packed = xh_old != nullptr;
    if (!u0 || !u2 || u0 == u2) return fail(TM_ERR_INVALID, "tm_heat_march2: needs distinct input/output fields");
    if (L.nghost < 2) return fail(TM_ERR_INVALID, "tm_heat_march2: needs nghost >= 2");
    if (ncomp_sweep < 1 || ncomp_sweep > L.ncomp) return fail(TM_ERR_INVALID, "tm_heat_march2: bad ncomp");
    if (strides_of(L).comp >= ((int64_t)1 << 32))
        return fail(TM_ERR_INVALID, "tm_heat_march2: one component of a slot must hold < 2^32 doubles");
    if (p->ncols == 0) return TM_OK;
    if (!p->even || p->max_nx > 64 || p->max_ny > 16)
        return fail(TM_ERR_INVALID, "tm_heat_march2: columns must be even-sized, <= 64 wide and <= 16 rows");
    March2Args a{};
    a.cols = p->d_cols;
    a.segs = p->d_segs;
    a.seg_begin = p->d_seg_begin;
    a.out = u2;
    a.L = L;
    a.c0 = dxi0;
    a.c1 = dxi1;
    a.c2 = dxi2;
    a.c3 = dtD;
    a.box_x = packed ? p->max_nx : p->max_nx + 4;
    a.box_y = p->max_ny + 4;
    a.xh_off = ((a.box_x * a.box_y + 15) / 16) * 16;
    // TMA destinations must be 128-B aligned: every slice starts on 16 doubles
    a.xh1_off = a.xh_off + ((2 * a.box_y + 15) / 16) * 16;
    a.stage_elems = packed ? a.xh1_off + ((2 * a.box_y + 15) / 16) * 16 : a.xh_off;
    a.u1_x = p->max_nx + 4;
    a.u1_elems = ((a.u1_x * (p->max_ny + 2) + 15) / 16) * 16;
    a.nbr27 = d_nbr27;
    a.xh_new = xh_new;
    a.nxb = p->max_nx;
    a.nyb = L.ny - 2 * L.nghost;
    a.nzb = L.nz - 2 * L.nghost;
    const size_t smem = ((size_t)kStages2 * a.stage_elems + (size_t)kU1Slots * a.u1_elems) * sizeof(double) +
                        kStages2 * sizeof(uint64_t);
    CUtensorMap map, xmap;
    rc = encode_plane_map(&map, L, u0, a.box_x, a.box_y);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    if (packed || d_nbr27) {
        if (a.nyb < 4 || a.nzb < 4 || a.nxb < 8 || a.nxb % 8)
            return fail(TM_ERR_INVALID, "tm_heat_march2: fused halos need box width % 8 == 0 and y, z extents >= 4");
        if (!d_nbr27) return fail(TM_ERR_INVALID, "tm_heat_march2: fused halos need the neighbour table");
    }
    if (packed) {
        // x halos as (2*(ny+4) doubles of a plane-side, 2*(nz+4) plane-sides, 1, slot*ncomp):
        // a column's rows are one contiguous 2*box_y run
        tm_layout X{};
        X.nslots = L.nslots;
        X.ncomp = L.ncomp;
        X.pitch = 2 * (a.nyb + 4);
        X.ny = 2 * (a.nzb + 4);
        X.nz = 1;
        rc = encode_plane_map(&xmap, X, xh_old, 2 * a.box_y, 1);
        if (rc) return rc;
        return launch_mode<1>(map, xmap, a, p, ncomp_sweep, smem, s);
    }
    xmap = map;
    if (d_nbr27) return launch_mode<2>(map, xmap, a, p, ncomp_sweep, smem, s);
    return launch_mode<0>(map, xmap, a, p, ncomp_sweep, smem, s);
}

}  // extern "C"
