// Kernel A2: persistent column-march heat sweep.
//
// Why: on B200 the halo rows/planes that neighbouring tile-CTAs share are not
// served from L2 (profiles/l2_experiments_r01.md) -- a 64x8x8 tile re-reads
// 1.65x its bytes from DRAM.  Here each CTA owns whole tile *columns* (the
// full z extent of a box's x-y tile) and marches through them, so every plane
// of the column is read once and the z halo costs 2 planes per column, not 2
// per tile.  The grid is persistent (a few CTAs per SM); CTA i takes a
// contiguous, equal share of all column planes, split into segments, and the
// TMA ring keeps streaming across segment boundaries.
//
// Two halo sources for x:
//   STD    -- the x ghost cells in the rows (same layout as Kernel A);
//   PACKED -- a packed x-halo buffer xh[slot*ncomp+c][z][side][y] (dense), so
//             rows are loaded exactly [x0, x0+nx) and the two ghost columns
//             cost 16 B per row instead of two 64-B DRAM blocks.
// With SCATTER the epilogue also writes each box's boundary values into its
// face neighbours' halos of the NEW field (y/z ghost rows/planes of unew and
// the packed x halo xh_new), so the next step needs no FillBoundary for
// intra-GPU neighbours.  The 7-point stencil needs face
// halos only; edge/corner ghosts are not touched on this path.
//
// Arithmetic is identical to Kernel A (reference flux form, FMA-free).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "tm_march_plan.cuh"

namespace {

using tmk::Segment;

// TMA ring depth (powers of two: stage and phase come from the plane counter by mask/shift).
// (8 heat stages measured: C2 62.6 us vs 56.9 us at 4 -- fewer CTAs fit; C3/C5 within +-3 %.)
constexpr int kHeatStages = 4;
constexpr int kGsrbStages = 4;

struct MarchArgs {
    const tm_block *cols;
    const Segment *segs;
    const int32_t *seg_begin;  // per CTA: segments [seg_begin[i], seg_begin[i+1])
    double *out;
    tm_layout L;
    double c0, c1, c2, c3;
    int32_t box_x, box_y, stage_elems;  // plane box (doubles) and stage stride
    int32_t xh_off;                     // offset of the x-halo slice inside a stage (PACKED)
    int32_t nyv, nzv;                   // packed x-halo extents (valid y, z of a slot)
    double *xh_new;                     // SCATTER: packed x halo of the new field
    double *gw;                         // GW: uold's storage, whose face ghosts the step fills
    const int32_t *nbr;                 // SCATTER: 6 neighbour slots per slot (-x,+x,-y,+y,-z,+z)
    const int64_t *fcells;              // FILL: (dst, src) element offsets in uold (edge/corner ghosts)
    int64_t nfcells;
    const CUtensorMap *pmaps;           // NBRH peer faces: [TM_MAX_PEERS][2] maps of the peer set (or null)
};

// Plane sequence of a CTA: for each of its segments, planes k0-1 .. k1 (k1-k0+2 planes).
struct PlaneCursor {
    int seg, q;  // segment index (absolute) and plane index within the segment
};

template <bool PACKED>
__device__ __forceinline__ void issue(const CUtensorMap *map, const CUtensorMap *xmap, const MarchArgs &a,
                                      double *stage, uint64_t *bar, const tm_block &c, int comp, int z,
                                      uint32_t tx_bytes) {
    using namespace tmk;
    const int w = c.slot * a.L.ncomp + comp;
    mbar_arrive_expect_tx(bar, tx_bytes);
    if (PACKED) {
        tma_load_plane(stage, map, bar, c.x0, c.y0 - 1, z, w);
        // x halo: y range of the column, both sides, valid plane z - nghost
        const int g = a.L.nghost;
        tma_load_plane(stage + a.xh_off, xmap, bar, c.y0 - g, 0, z - g, w);
    } else {
        tma_load_plane(stage, map, bar, (c.x0 - 1) & ~1, c.y0 - 1, z, w);
    }
}

// One plane as a consumer warp needs it: its RPW rows of CPL cells per lane
// and their in-plane flux sums.
template <int CPL, int RPW, bool HS>
struct PlaneRegs {
    double u[RPW][CPL];                        // the warp's cells
    double hs[HS ? RPW : 1][HS ? CPL : 1];     // their in-plane flux sums (x and y parts)
};

// NBRH (fused mode, uniform columns): the z halo planes and the y halo rows at
// box faces are read straight from the face neighbour's valid cells in uold
// (the same values a FillBoundary would have copied into our ghosts), so the
// step never writes y/z face ghosts of unew.  Faces whose neighbour is on
// another rank (or none) still come from our own ghost cells, which the halo
// exchange fills.  Stage rows: 0 = y0-1 (1-row box), 1..ny = the column
// (ny-row box), ny+1 = y0+ny (1-row box); then the packed x halo.
struct NbrFaces {
    int32_t ylo, yhi, zlo, zhi;  // neighbour slot per face, < 0: use our own ghosts
    bool top, bot;               // the column's first / last row is a box face
};

// A face's source: local slot v >= 0 (the field's own maps) or a peer face v <= -3
// (TM_NBR_PEER: slot of peer p, read through peer p's maps over NVLink); -1 / -2 (none,
// remote via the halo exchange): no source, the halo comes from our own ghost cells.
__device__ __forceinline__ bool nbr_src(int32_t v, const MarchArgs &a, const CUtensorMap *map,
                                        const CUtensorMap *rmap, int &slot, const CUtensorMap *&m,
                                        const CUtensorMap *&r) {
    if (v >= 0) {
        slot = v;
        m = map;
        r = rmap;
        return true;
    }
    if (v <= -3) {
        const int q = -3 - v;
        slot = q & 0xffffff;
        m = a.pmaps + 2 * (q >> 24);
        r = m + 1;
        return true;
    }
    return false;
}

__device__ __forceinline__ void issue_nbr(const CUtensorMap *map, const CUtensorMap *rmap, const CUtensorMap *xmap,
                                          const MarchArgs &a, double *stage, uint64_t *bar, const tm_block &c,
                                          const NbrFaces &f, int comp, int z, uint32_t tx_bytes) {
    using namespace tmk;
    const int nc = a.L.ncomp, g = a.L.nghost;
    const int w = c.slot * nc + comp;
    const int zl = z - g;  // valid z index of the plane
    int ws = w, zs = z, s = 0;
    const CUtensorMap *zm = map, *zr = rmap, *m = map, *r = rmap;
    if (zl < 0 && nbr_src(f.zlo, a, map, rmap, s, m, r)) {
        ws = s * nc + comp;
        zs = z + a.nzv;
        zm = m;
        zr = r;
    } else if (zl >= a.nzv && nbr_src(f.zhi, a, map, rmap, s, m, r)) {
        ws = s * nc + comp;
        zs = z - a.nzv;
        zm = m;
        zr = r;
    }
    const bool centre = zl >= 0 && zl < a.nzv;  // halo planes: only their column rows are used
    mbar_arrive_expect_tx(bar, tx_bytes);
    const int bx = a.box_x;
    tma_load_plane(stage + bx, zm, bar, c.x0, c.y0, zs, ws);
    if (centre && f.top && nbr_src(f.ylo, a, map, rmap, s, m, r))
        tma_load_plane(stage, r, bar, c.x0, c.y0 - 1 + a.nyv, zs, s * nc + comp);
    else
        tma_load_plane(stage, zr, bar, c.x0, c.y0 - 1, zs, ws);
    if (centre && f.bot && nbr_src(f.yhi, a, map, rmap, s, m, r))
        tma_load_plane(stage + (c.ny + 1) * bx, r, bar, c.x0, c.y0 + c.ny - a.nyv, zs, s * nc + comp);
    else
        tma_load_plane(stage + (c.ny + 1) * bx, zr, bar, c.x0, c.y0 + c.ny, zs, ws);
    tma_load_plane(stage + a.xh_off, xmap, bar, c.y0 - g, 0, z - g, w);
}

// Warp-specialised pipeline: warps 0..NWARP-1 compute, warp NWARP is the TMA
// producer.  full[s] completes when stage s holds its plane (TMA transaction
// bytes); empty[s] completes when all NWARP consumer warps released it.  No
// CTA-wide barrier in the steady state: fast warps run ahead up to the ring
// depth while the producer refills each stage as soon as it is free.
// GW (TM_HALO_FUSED_NBR_GHOSTS): the y/z halo rows and planes the neighbour-halo step loads
// are exactly the y/z face ghosts a FillBoundary of uold writes, so the step also stores them
// into uold's ghosts -- the deferred y/z part of the preceding fill_boundary
// (multifab.fill_boundary), at no extra read.  Other CTAs read only uold's valid cells.
// HW (half-warp rows, boxes 18..32 wide): lanes 0-15 and 16-31 march two different row groups
// of the column, 2 cells per lane, so a warp covers 2*RPW rows of a narrow box with the
// two-cells-per-lane instruction stream instead of one cell per lane (C5's 32-wide boxes:
// ~61 instructions per cell at one cell per lane against ~40 at two).
// FILL (with GW): one more warp runs the preceding FillBoundary's remaining tags on uold -- its
// edge/corner ghosts, which the 7-point sweep never reads -- while the other warps march, so the
// reference-shaped loop (fill_boundary; heat_step) needs no separate copy launch per step.
template <int CPL, int NWARP, int RPW, bool PACKED, bool SCATTER, bool REV, bool NBRH, bool GW = false,
          bool HW = false, bool FILL = false>
__global__ void __launch_bounds__((NWARP + 1 + FILL) * 32, NWARP <= 4 ? 3 : (NWARP <= 8 ? 2 : 1)) march_kernel(const __grid_constant__ CUtensorMap map,
                                                                 const __grid_constant__ CUtensorMap xmap,
                                                                 const __grid_constant__ CUtensorMap rmap,
                                                                 MarchArgs a) {
    static_assert(!NBRH || (PACKED && SCATTER), "neighbour-sourced halos belong to the fused mode");
    static_assert(!GW || (NBRH && !REV), "face-ghost writes ride on the forward neighbour-halo step");
    static_assert(!FILL || GW, "the fill warp rides on the face-ghost-writing step");
    // SCATTER: the epilogue writes the packed x halos of the new field (xh_new); with x halos
    // from the packed buffer and y/z halos from ghost cells (TM_HALO_FUSED_SCATTER) it also
    // writes the y/z face ghosts of unew.  TM_HALO_GHOSTS_XH (!PACKED) writes xh_new only.
    constexpr bool kYZ = SCATTER && PACKED && !NBRH;
    using namespace tmk;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kHeatStages * a.stage_elems * sizeof(double));
    uint64_t *empty = bars + kHeatStages;

    const int comp = blockIdx.y;
    const int s_begin = a.seg_begin[blockIdx.x], s_end = a.seg_begin[blockIdx.x + 1];
    if (s_begin >= s_end) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bx = a.box_x;
    const uint32_t tx_bytes =
        (uint32_t)((a.box_x * a.box_y + (PACKED ? 2 * (a.box_y - 2) : 0)) * (int)sizeof(double));

    if (tid == 0) {
        prefetch_tensormap(&map);
        if (PACKED) prefetch_tensormap(&xmap);
        if (NBRH) prefetch_tensormap(&rmap);
#pragma unroll
        for (int s = 0; s < kHeatStages; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&empty[s], NWARP);
        }
        fence_mbar_init();
    }
    grid_dep_launch();  // the next step's CTAs may take SM slots as ours retire
    __syncthreads();
    grid_dep_wait();  // previous step complete: its unew is our uold, its uold our unew

    if (FILL && warp == NWARP + 1) {  // ---------------- fill warp ----------------
        // one cell per lane: the edge/corner tags are thousands of one-cell rows (a z edge is
        // one task per plane in Kernel B's row tasks), so lanes take independent cells
        // (kB cells per lane per trip: every index and value load in flight before the stores)
        if (blockIdx.y == 0) {  // the list covers every component
            constexpr int kB = 8;
            const int64_t stride = (int64_t)gridDim.x * 32;
            for (int64_t i0 = (int64_t)blockIdx.x * 32 + lane; i0 < a.nfcells; i0 += kB * stride) {
                longlong2 ds[kB];
                double v[kB];
#pragma unroll
                for (int b = 0; b < kB; ++b) {
                    const int64_t i = i0 + b * stride;
                    ds[b] = i < a.nfcells ? reinterpret_cast<const longlong2 *>(a.fcells)[i] : make_longlong2(-1, 0);
                }
#pragma unroll
                for (int b = 0; b < kB; ++b) v[b] = ds[b].x >= 0 ? __ldg(a.gw + ds[b].y) : 0.0;
#pragma unroll
                for (int b = 0; b < kB; ++b)
                    if (ds[b].x >= 0) a.gw[ds[b].x] = v[b];
            }
        }
        return;
    }
    if (warp == NWARP) {  // ---------------- producer warp ----------------
        if (lane == 0) {
            int p = 0;
            for (int si = 0; si < s_end - s_begin; ++si) {
                const Segment sg = a.segs[REV ? s_end - 1 - si : s_begin + si];
                const tm_block c = a.cols[sg.col];
                const int n = sg.k1 - sg.k0 + 2;
                NbrFaces f{};
                if (NBRH) {
                    const int32_t *nb = a.nbr + 6 * c.slot;
                    f.ylo = nb[2];
                    f.yhi = nb[3];
                    f.zlo = nb[4];
                    f.zhi = nb[5];
                    f.top = c.y0 - a.L.nghost == 0;
                    f.bot = c.y0 - a.L.nghost + c.ny == a.nyv;
                }
                for (int q = 0; q < n; ++q, ++p) {
                    const int st_i = p % kHeatStages;
                    if (p >= kHeatStages) mbar_wait(&empty[st_i], ((p / kHeatStages) - 1) & 1);
                    const int z = REV ? c.z0 + sg.k1 - q : c.z0 + sg.k0 - 1 + q;
                    if (NBRH)
                        issue_nbr(&map, &rmap, &xmap, a, stages + st_i * a.stage_elems, &bars[st_i], c, f, comp, z,
                                  tx_bytes);
                    else
                        issue<PACKED>(&map, &xmap, a, stages + st_i * a.stage_elems, &bars[st_i], c, comp, z,
                                      tx_bytes);
                }
            }
        }
        return;
    }

    // ---------------- consumer warps ----------------
    // Hot-loop bookkeeping is kept to 32-bit offsets and running counters: the
    // plane loop is issue-bound as much as it is memory-bound (ncu: ~60% issue
    // active), so every per-plane integer instruction costs time.
    const uint32_t sbase = smem_u32(stages);
    const uint32_t bfull = smem_u32(bars), bempty = smem_u32(empty);
    const uint32_t sbytes = (uint32_t)a.stage_elems * 8u;
    auto saddr = [&](uint32_t q) { return sbase + (q & (kHeatStages - 1)) * sbytes; };
    auto wait_plane = [&](uint32_t q) { mbar_wait_u32(bfull + (q & (kHeatStages - 1)) * 8u, (q / kHeatStages) & 1u); };
    auto release = [&](uint32_t q) {
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bempty + (q & (kHeatStages - 1)) * 8u);
    };

    const double c0 = a.c0, c1 = a.c1, c2 = a.c2, c3 = a.c3;
    const Strides st = strides_of(a.L);
    const int g_ng = a.L.nghost;
    const int xsh = PACKED ? 0 : 2;  // smem column of a column's first cell (x0 is even)
    const int max_ny = a.box_y - 2;
    const uint32_t ystep = (uint32_t)bx * 8u;
    const uint32_t pstep = (uint32_t)st.plane;  // < 2^31 (host-checked)
    const int nyb = a.nyv, nzb = a.nzv;
    uint32_t g = 0;  // CTA-wide plane counter of the current segment's first plane

    // REV: segments in reverse order and each column marched downward in z, so a
    // step that follows a forward step first reads the planes that step wrote
    // last (still in L2).  Same fluxes, same bits.
    for (int si = 0; si < s_end - s_begin; ++si) {
        const Segment sg = a.segs[REV ? s_end - 1 - si : s_begin + si];
        const tm_block c = a.cols[sg.col];
        const int nk = sg.k1 - sg.k0;
        // this lane's position: x slot lx within its row group, first row row0 of the group
        const int lx = HW ? (lane & 15) : lane;
        const int row0 = HW ? warp * 2 * RPW + (lane >> 4) * RPW : warp * RPW;
        const int xi = min(lx * CPL, c.nx - CPL);  // lane's first cell (clamped for idle lanes)
        const bool lane_on = lx * CPL < c.nx;
        // output rows: 64-bit row bases + one 32-bit running plane offset
        double *const obase = a.out + (int64_t)c.slot * st.slot + (int64_t)comp * st.comp;
        uint32_t koff = (uint32_t)((int64_t)(c.z0 + sg.k0 + (REV ? nk - 1 : 0)) * st.plane + (int64_t)c.y0 * st.row +
                                   c.x0 + xi);
        double *orow[RPW];
        bool on[RPW];
        uint32_t roff[RPW];  // smem byte offset of the row's first cell (rows past max_ny clamp; never stored)
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int r = row0 + i;
            on[i] = lane_on && r < c.ny;
            orow[i] = obase + (int64_t)r * st.row;
            roff[i] = (uint32_t)((min(r, max_ny) + 1) * bx + xi + xsh) * 8u;
        }
        // the row after this warp's last row (its y+1 neighbours): clamped to the stage's last
        // row for warps whose rows all lie past the column (values never stored)
        const uint32_t ypo = (uint32_t)((min(row0 + RPW - 1, max_ny - 1) + 2) * bx + xi + xsh) * 8u;
        uint32_t xlo[RPW], xro[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int r = min(row0 + i, c.ny - 1);
            const bool left_edge = PACKED && lx == 0;
            const bool right_edge = PACKED && (xi + CPL == c.nx);
            xlo[i] = left_edge ? (uint32_t)(a.xh_off + r) * 8u : roff[i] - 8u;
            xro[i] = right_edge ? (uint32_t)(a.xh_off + max_ny + r) * 8u : roff[i] + (uint32_t)CPL * 8u;
        }
        // SCATTER targets.  y: only the column's first row (-y face) and last row (+y face)
        // can be box faces; z: two planes of the column, warp-uniform; x: the lanes holding
        // x = 0 / x = nx-1 write the neighbour's packed halo (consecutive y, one plane apart).
        const int32_t *nb = a.nbr + 6 * c.slot;
        const int zl0 = c.z0 - g_ng + sg.k0;  // valid z index of the segment's first plane
        const int yl0 = c.y0 - g_ng;          // valid y index of the column's first row
        int ylo_i = -1, yhi_i = -1;
        double *ylo = nullptr, *yhi = nullptr;
        double *xhp = nullptr;
        bool x_right = false;
        int kz_lo = -1, kz_hi = -1;
        int64_t zoff_lo = 0, zoff_hi = 0;
        if (SCATTER) {
            if (kYZ && row0 == 0 && yl0 == 0 && nb[2] >= 0 && on[0]) {
                ylo_i = 0;
                ylo = orow[0] + (int64_t)(nb[2] - c.slot) * st.slot + (int64_t)nyb * st.row;
            }
            const int rl = c.ny - 1;  // last row of the column
            if (kYZ && yl0 + c.ny == nyb && nb[3] >= 0 && rl >= row0 && rl < row0 + RPW && lane_on) {
                yhi_i = rl - row0;
                yhi = obase + (int64_t)rl * st.row + (int64_t)(nb[3] - c.slot) * st.slot - (int64_t)nyb * st.row;
            }
            const int xl0 = c.x0 - a.L.xoff + lx * CPL;
            if (lane_on && xl0 == 0 && nb[0] >= 0)  // our x = 0 cells -> the -x neighbour's right halo
                xhp = a.xh_new + (((int64_t)(nb[0] * a.L.ncomp + comp) * nzb + zl0) * 2 + 1) * nyb + yl0 + row0;
            if (lane_on && xl0 + CPL == c.nx && nb[1] >= 0) {
                xhp = a.xh_new + (((int64_t)(nb[1] * a.L.ncomp + comp) * nzb + zl0) * 2 + 0) * nyb + yl0 + row0;
                x_right = true;
            }
            if (kYZ && nb[4] >= 0 && zl0 <= 0 && 0 < zl0 + nk) {
                kz_lo = -zl0;
                zoff_lo = (int64_t)(nb[4] - c.slot) * st.slot + (int64_t)nzb * st.plane;
            }
            if (kYZ && nb[5] >= 0 && zl0 <= nzb - 1 && nzb - 1 < zl0 + nk) {
                kz_hi = nzb - 1 - zl0;
                zoff_hi = (int64_t)(nb[5] - c.slot) * st.slot - (int64_t)nzb * st.plane;
            }
        }
        const int64_t xstep = REV ? -2 * (int64_t)nyb : 2 * (int64_t)nyb;
        if (REV && xhp) xhp += (int64_t)(nk - 1) * 2 * nyb;  // x halo of the first plane processed
        // RPW == 2: rows come in pairs (even column heights), so on[0] == on[1]
        const bool xh_on = xhp != nullptr && on[0];
        uint64_t xh_addr = reinterpret_cast<uint64_t>(xhp);
        // GW targets (uold's y/z face ghosts, faces with a local neighbour only): the y ghost row
        // above / below the column by the warp holding its first / last row, the z ghost planes
        // from the priming / last halo plane.  (x faces: the packed halos ARE those ghosts; the
        // host keeps them as a snapshot instead of scattering 8-B values over every row.)
        double *gbase = nullptr;
        bool gy_lo = false, gy_hi = false, gz_lo = false, gz_hi = false;
        if (GW) {
            // koff addresses the column's first row: this lane's rows start row0 rows below
            gbase = a.gw + (int64_t)c.slot * st.slot + (int64_t)comp * st.comp + (int64_t)row0 * st.row;
            gy_lo = lane_on && row0 == 0 && yl0 == 0 && nb[2] >= 0;
            gy_hi = lane_on && row0 + RPW - 1 == c.ny - 1 && yl0 + c.ny == nyb && nb[3] >= 0;
            gz_lo = zl0 == 0 && nb[4] >= 0;
            gz_hi = zl0 + nk == nzb && nb[5] >= 0;
        }

        // priming: planes k0-1 and k0 -> carried z flux and centre values
        // Early release (kEarly, instances whose registers allow it): when a plane lands, the
        // warp reads everything it needs from it -- its rows, the rows just above and below,
        // the x neighbours of its row ends -- computes the plane's in-plane flux sums
        // hs = (fx+ - fx-)*dxi0 + (fy+ - fy-)*dxi1 (the first half of the reference's sum,
        // same operation order), and hands the stage back at once: every stage but the one
        // being read stays in flight.  Every loaded value is consumed by that arithmetic
        // before the release, so the stage is never overwritten under an outstanding read.
        // Otherwise the centre plane's stage is held through the arithmetic (half the ring in
        // flight).
        constexpr bool kEarly = CPL * RPW <= 4;
        PlaneRegs<CPL, RPW, kEarly> pa, pb;
        double fzm[RPW][CPL];
        auto load_u = [&](uint32_t sb, PlaneRegs<CPL, RPW, kEarly> &P) {
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
#pragma unroll
                for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                    if constexpr (CPL >= 2)
                        lds_f64x2(sb + roff[i] + 8u * j, P.u[i][j], P.u[i][j + 1]);
                    else
                        P.u[i][j] = lds_f64(sb + roff[i] + 8u * j);
                }
            }
        };
        // in-plane flux sums of plane sb for the warp's cells (y fluxes between consecutive
        // rows are shared by the two rows; x fluxes between a lane's cells shared likewise)
        auto inplane = [&](uint32_t sb, const double (&u)[RPW][CPL], double (&hs)[RPW][CPL], uint32_t goff,
                           bool centre) {
            double ym[CPL], yp[CPL];
#pragma unroll
            for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                if constexpr (CPL >= 2) {
                    lds_f64x2(sb + roff[0] - ystep + 8u * j, ym[j], ym[j + 1]);
                    lds_f64x2(sb + ypo + 8u * j, yp[j], yp[j + 1]);
                } else {
                    ym[j] = lds_f64(sb + roff[0] - ystep + 8u * j);
                    yp[j] = lds_f64(sb + ypo + 8u * j);
                }
            }
            if (GW && centre) {
                if (gy_lo) {
#pragma unroll
                    for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                        double *d = gbase + goff - st.row + j;
                        if constexpr (CPL >= 2)
                            *reinterpret_cast<double2 *>(d) = make_double2(ym[j], ym[j + 1]);
                        else
                            *d = ym[j];
                    }
                }
                if (gy_hi) {
#pragma unroll
                    for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                        double *d = gbase + goff + RPW * st.row + j;
                        if constexpr (CPL >= 2)
                            *reinterpret_cast<double2 *>(d) = make_double2(yp[j], yp[j + 1]);
                        else
                            *d = yp[j];
                    }
                }
            }
            double fy[RPW + 1][CPL];
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
                fy[0][j] = rn_mul(rn_sub(u[0][j], ym[j]), c1);
#pragma unroll
                for (int i = 1; i < RPW; ++i) fy[i][j] = rn_mul(rn_sub(u[i][j], u[i - 1][j]), c1);
                fy[RPW][j] = rn_mul(rn_sub(yp[j], u[RPW - 1][j]), c1);
            }
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                const double xl = lds_f64(sb + xlo[i]);
                const double xr = lds_f64(sb + xro[i]);
                double fx[CPL + 1];
                fx[0] = rn_mul(rn_sub(u[i][0], xl), c0);
#pragma unroll
                for (int j = 1; j < CPL; ++j) fx[j] = rn_mul(rn_sub(u[i][j], u[i][j - 1]), c0);
                fx[CPL] = rn_mul(rn_sub(xr, u[i][CPL - 1]), c0);
#pragma unroll
                for (int j = 0; j < CPL; ++j)
                    hs[i][j] = rn_add(rn_mul(rn_sub(fx[j + 1], fx[j]), c0), rn_mul(rn_sub(fy[i + 1][j], fy[i][j]), c1));
            }
        };
        auto fetch = [&](uint32_t q, PlaneRegs<CPL, RPW, kEarly> &P, uint32_t goff, bool centre) {
            wait_plane(q);
            const uint32_t sb = saddr(q);
            load_u(sb, P);
            if constexpr (kEarly) {
                double(&hs)[RPW][CPL] = P.hs;
                inplane(sb, P.u, hs, goff, centre);
                release(q);
            }
        };
        // z ghost planes of uold (GW): the rows of the plane below the box / above it, as loaded
        auto st_zghost = [&](const double (&v)[RPW][CPL], uint32_t goff) {
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                if (!on[i]) continue;
#pragma unroll
                for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                    double *d = gbase + goff + i * st.row + j;
                    if constexpr (CPL >= 2)
                        *reinterpret_cast<double2 *>(d) = make_double2(v[i][j], v[i][j + 1]);
                    else
                        *d = v[i][j];
                }
            }
        };
        {
            // priming: plane k0-1 (forward; k1 reversed) for the carried z flux, then plane k0
            wait_plane(g);
            const uint32_t s0 = saddr(g);
            double lo[RPW][CPL];
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; ++j) lo[i][j] = lds_f64(s0 + roff[i] + 8u * j);
            fetch(g + 1, pa, koff, true);
            if (GW && gz_lo) st_zghost(lo, koff - pstep);
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; ++j)  // u[k+1] - u[k] in either direction
                    fzm[i][j] = REV ? rn_mul(rn_sub(lo[i][j], pa.u[i][j]), c2) : rn_mul(rn_sub(pa.u[i][j], lo[i][j]), c2);
            release(g);  // after lo[][] has been consumed
        }
        // one plane: centre values in cur, the next plane lands in nxt
        auto plane = [&](int kk, PlaneRegs<CPL, RPW, kEarly> &cur, PlaneRegs<CPL, RPW, kEarly> &nxt) {
            const uint32_t gc = g + 1 + (uint32_t)kk;
            double hsl[RPW][CPL];  // non-early instances: the centre plane's flux sums, computed here
            if constexpr (!kEarly) inplane(saddr(gc), cur.u, hsl, koff, true);
            const uint32_t knext = REV ? koff - pstep : koff + pstep;
            fetch(gc + 1, nxt, knext, kk + 1 < nk);
            if (GW && gz_hi && kk == nk - 1) st_zghost(nxt.u, knext);
            double out[RPW][CPL];
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    const double u0 = cur.u[i][j];
                    // fresh z flux toward the next plane; fzm[][] carries the other one
                    const double fnew =
                        REV ? rn_mul(rn_sub(u0, nxt.u[i][j]), c2) : rn_mul(rn_sub(nxt.u[i][j], u0), c2);
                    const double fzp = REV ? fzm[i][j] : fnew, fzn = REV ? fnew : fzm[i][j];
                    double hs;
                    if constexpr (kEarly)
                        hs = cur.hs[i][j];
                    else
                        hs = hsl[i][j];
                    const double sum = rn_add(hs, rn_mul(rn_sub(fzp, fzn), c2));
                    out[i][j] = rn_add(u0, rn_mul(c3, sum));
                    fzm[i][j] = fnew;
                }
            }
            if constexpr (!kEarly) release(gc);  // all shared reads of the centre plane are done
            auto st_cells = [&](double *d, int i) {
#pragma unroll
                for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                    if constexpr (CPL >= 2)
                        *reinterpret_cast<double2 *>(d + j) = make_double2(out[i][j], out[i][j + 1]);
                    else
                        d[j] = out[i][j];
                }
            };
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                if (!on[i]) continue;
                st_cells(orow[i] + koff, i);
                if (kYZ) {
                    if (i == ylo_i) st_cells(ylo + koff, i);
                    if (i == yhi_i) st_cells(yhi + koff, i);
                }
            }
            if (SCATTER) {
                const int kz = REV ? nk - 1 - kk : kk;  // plane index from k0
                if (kYZ && (kz == kz_lo || kz == kz_hi)) {  // warp-uniform, two planes per column
                    const int64_t zd = kz == kz_lo ? zoff_lo : zoff_hi;
#pragma unroll
                    for (int i = 0; i < RPW; ++i)
                        if (on[i]) st_cells(orow[i] + koff + zd, i);
                }
                if constexpr (RPW == 2) {
                    // lanes 0 / 31 of the box's x faces: one predicated 16-B store of the warp's two
                    // rows (consecutive y in the packed halo), no divergent branch in the plane loop
                    st_global_f64x2_if(xh_addr, x_right ? out[0][CPL - 1] : out[0][0],
                                       x_right ? out[1][CPL - 1] : out[1][0], xh_on);
                    xh_addr += (uint64_t)(xstep * 8);
                } else if (xhp) {
#pragma unroll
                    for (int i = 0; i < RPW; ++i)
                        if (on[i]) xhp[i] = x_right ? out[i][CPL - 1] : out[i][0];
                    xhp += xstep;
                }
            }
            koff = REV ? koff - pstep : koff + pstep;
        };
        int kk = 0;
        for (; kk + 1 < nk; kk += 2) {  // ping-pong: no register rotation
            plane(kk, pa, pb);
            plane(kk + 1, pb, pa);
        }
        if (kk < nk) plane(kk, pa, pb);
        if constexpr (!kEarly) release(g + nk + 1);
        g += nk + 2;
    }
}


// ---------------------------------------------------------------------------
// Fused red-black Gauss-Seidel colour pass on the same column march.
//
// In place on phi: a pass updates only cells of one colour, and every value it
// reads (x/y/z neighbours) has the other colour, so no CTA ever reads a value
// another CTA writes in the same pass -- including the halo rows/planes of
// neighbouring columns and the ghosts it scatters into (colour-c values into
// ghost cells that this pass reads only at colour 1-c).  Each lane stores its
// cell pair with double2 (the unchanged cell re-written with the bits it
// already holds).  The stage holds [phi plane + y halo][packed x halo][rhs rows].
// Per-cell form (builder-owned, oracle/tm_oracle.c orc_gsrb_color):
//   s = ((((w + e) + s_) + n) + b) + t ;  phi = (s + h2*rhs) / 6
// ---------------------------------------------------------------------------
struct GsrbArgs {
    MarchArgs m;        // columns, segments, phi (out), layout, xh scatter, nbr, box, stage
    tm_layout R;        // rhs layout
    int32_t rhs_off;    // offset of the rhs slice inside a stage (doubles)
    int32_t color;
    double h2;
};

template <int CPL, int NWARP, int RPW>
__global__ void __launch_bounds__((NWARP + 1) * 32, NWARP <= 4 ? 3 : (NWARP <= 8 ? 2 : 1))
gsrb_march_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap xmap,
                  const __grid_constant__ CUtensorMap rmap, GsrbArgs ga) {
    using namespace tmk;
    const MarchArgs &a = ga.m;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kGsrbStages * a.stage_elems * sizeof(double));
    uint64_t *empty = bars + kGsrbStages;

    const int s_begin = a.seg_begin[blockIdx.x], s_end = a.seg_begin[blockIdx.x + 1];
    if (s_begin >= s_end) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bx = a.box_x;
    const int ny_box = a.box_y - 2;
    const uint32_t tx_bytes = (uint32_t)((a.box_x * a.box_y + 2 * ny_box + a.box_x * ny_box) * (int)sizeof(double));
    const int g_ng = a.L.nghost;

    if (tid == 0) {
        prefetch_tensormap(&map);
        prefetch_tensormap(&xmap);
        prefetch_tensormap(&rmap);
#pragma unroll
        for (int s = 0; s < kGsrbStages; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&empty[s], NWARP);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NWARP) {  // producer
        if (lane == 0) {
            int p = 0;
            for (int s = s_begin; s < s_end; ++s) {
                const Segment sg = a.segs[s];
                const tm_block c = a.cols[sg.col];
                const int w = c.slot;  // ncomp == 1
                const int n = sg.k1 - sg.k0 + 2;
                for (int q = 0; q < n; ++q, ++p) {
                    const int st_i = p % kGsrbStages;
                    if (p >= kGsrbStages) mbar_wait(&empty[st_i], ((p / kGsrbStages) - 1) & 1);
                    double *stage = stages + st_i * a.stage_elems;
                    const int z = c.z0 + sg.k0 - 1 + q;
                    mbar_arrive_expect_tx(&bars[st_i], tx_bytes);
                    tma_load_plane(stage, &map, &bars[st_i], c.x0, c.y0 - 1, z, w);
                    tma_load_plane(stage + a.xh_off, &xmap, &bars[st_i], c.y0 - g_ng, 0, z - g_ng, w);
                    tma_load_plane(stage + ga.rhs_off, &rmap, &bars[st_i], c.x0 - a.L.xoff + ga.R.xoff,
                                   c.y0 - g_ng + ga.R.nghost, z - g_ng + ga.R.nghost, w);
                }
            }
        }
        return;
    }

    const uint32_t sbase = smem_u32(stages);
    const uint32_t bfull = smem_u32(bars), bempty = smem_u32(empty);
    const uint32_t sbytes = (uint32_t)a.stage_elems * 8u;
    auto saddr = [&](uint32_t q) { return sbase + (q & (kGsrbStages - 1)) * sbytes; };
    auto wait_plane = [&](uint32_t q) { mbar_wait_u32(bfull + (q & (kGsrbStages - 1)) * 8u, (q / kGsrbStages) & 1u); };
    auto release = [&](uint32_t q) {
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bempty + (q & (kGsrbStages - 1)) * 8u);
    };
    const Strides st = strides_of(a.L);
    const double h2 = ga.h2;
    const uint32_t ystep = (uint32_t)bx * 8u;
    const uint32_t pstep = (uint32_t)st.plane;  // < 2^31 (host-checked)
    const int nyb = a.nyv, nzb = a.nzv;
    uint32_t g = 0;
    for (int s = s_begin; s < s_end; ++s) {
        const Segment sg = a.segs[s];
        const tm_block c = a.cols[sg.col];
        const int nk = sg.k1 - sg.k0;
        const int32_t *nb = a.nbr + 6 * c.slot;
        const int zl0 = c.z0 - g_ng + sg.k0;
        const int yl0 = c.y0 - g_ng;
        const bool lane_on = lane * CPL < c.nx;
        const int xc = min(lane * CPL, c.nx - CPL);
        double *const obase = a.out + (int64_t)c.slot * st.slot;  // ncomp == 1
        uint32_t koff = (uint32_t)((int64_t)(c.z0 + sg.k0) * st.plane + (int64_t)c.y0 * st.row + c.x0 + xc);
        uint32_t roff[RPW], xlo[RPW], xro[RPW], rof[RPW];
        bool on[RPW];
        double *orow[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int r = warp * RPW + i;
            const int rc = min(r, c.ny - 1);
            on[i] = lane_on && r < c.ny;
            orow[i] = obase + (int64_t)r * st.row;
            roff[i] = (uint32_t)((min(r, ny_box) + 1) * bx + xc) * 8u;  // rows past ny_box clamp; never stored
            xlo[i] = (lane == 0) ? (uint32_t)(a.xh_off + rc) * 8u : roff[i] - 8u;
            xro[i] = (xc + CPL == c.nx) ? (uint32_t)(a.xh_off + ny_box + rc) * 8u : roff[i] + (uint32_t)CPL * 8u;
            rof[i] = (uint32_t)(ga.rhs_off + min(r, ny_box - 1) * bx + xc) * 8u;
        }
        // y+1 row of this warp's last row, clamped inside the stage (see march_kernel)
        const uint32_t ypo = (uint32_t)((min(warp * RPW + RPW - 1, ny_box - 1) + 2) * bx + xc) * 8u;
        // colour of this lane's cell 0 in row 0 at plane k0, flipped per row and per plane
        const int par0 = (c.parity + xc + warp * RPW + sg.k0 + ga.color) & 1;
        // scatter targets (see march_kernel)
        int ylo_i = -1, yhi_i = -1;
        double *ylo = nullptr, *yhi = nullptr, *xhp = nullptr;
        bool x_right = false;
        if (warp == 0 && yl0 == 0 && nb[2] >= 0 && on[0]) {
            ylo_i = 0;
            ylo = orow[0] + (int64_t)(nb[2] - c.slot) * st.slot + (int64_t)nyb * st.row;
        }
        {
            const int rl = c.ny - 1;
            if (yl0 + c.ny == nyb && nb[3] >= 0 && rl / RPW == warp && lane_on) {
                yhi_i = rl % RPW;
                yhi = obase + (int64_t)rl * st.row + (int64_t)(nb[3] - c.slot) * st.slot - (int64_t)nyb * st.row;
            }
        }
        const int xl0 = c.x0 - a.L.xoff + xc;
        if (lane_on && xl0 == 0 && nb[0] >= 0)
            xhp = a.xh_new + ((int64_t)(nb[0] * nzb + zl0) * 2 + 1) * nyb + yl0 + warp * RPW;
        if (lane_on && xl0 + CPL == c.nx && nb[1] >= 0) {
            xhp = a.xh_new + ((int64_t)(nb[1] * nzb + zl0) * 2 + 0) * nyb + yl0 + warp * RPW;
            x_right = true;
        }
        int kz_lo = -1, kz_hi = -1;
        int64_t zoff_lo = 0, zoff_hi = 0;
        if (nb[4] >= 0 && zl0 <= 0 && 0 < zl0 + nk) {
            kz_lo = -zl0;
            zoff_lo = (int64_t)(nb[4] - c.slot) * st.slot + (int64_t)nzb * st.plane;
        }
        if (nb[5] >= 0 && zl0 <= nzb - 1 && nzb - 1 < zl0 + nk) {
            kz_hi = nzb - 1 - zl0;
            zoff_hi = (int64_t)(nb[5] - c.slot) * st.slot - (int64_t)nzb * st.plane;
        }
        const uint32_t xstep = 2u * (uint32_t)nyb;
        uint32_t xk = 0;

        double um[RPW][CPL], uc[RPW][CPL];
        wait_plane(g);
        wait_plane(g + 1);
        {
            const uint32_t s0 = saddr(g), s1 = saddr(g + 1);
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    um[i][j] = lds_f64(s0 + roff[i] + 8u * j);
                    uc[i][j] = lds_f64(s1 + roff[i] + 8u * j);
                }
        }
        release(g);
        for (int kk = 0; kk < nk; ++kk) {
            const uint32_t gc = g + 1 + (uint32_t)kk;
            const uint32_t sc = saddr(gc), sn = saddr(gc + 1);
            wait_plane(gc + 1);
            double out[RPW][CPL], un[RPW][CPL];
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                    if constexpr (CPL >= 2)
                        lds_f64x2(sn + roff[i] + 8u * j, un[i][j], un[i][j + 1]);
                    else
                        un[i][j] = lds_f64(sn + roff[i] + 8u * j);
                }
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                // p: offset of the updated cell inside each cell pair (CPL >= 2); for CPL == 1
                // the lane's single cell is updated iff p == 0.  Neighbours x+-1 of an updated
                // cell are this lane's other-colour cells or the row's x halo.
                const int p = (par0 + i + kk) & 1;
                if constexpr (CPL == 1) {
                    const double xl = lds_f64(sc + xlo[i]), xr = lds_f64(sc + xro[i]);
                    const double ym = i > 0 ? uc[i - 1][0] : lds_f64(sc + roff[0] - ystep);
                    const double yp = i < RPW - 1 ? uc[i + 1][0] : lds_f64(sc + ypo);
                    const double rh = lds_f64(sc + rof[i]);
                    double sum = rn_add(rn_add(rn_add(rn_add(rn_add(xl, xr), ym), yp), um[i][0]), un[i][0]);
                    const double upd = __ddiv_rn(rn_add(sum, rn_mul(h2, rh)), 6.0);
                    out[i][0] = p == 0 ? upd : uc[i][0];
                } else {
                    const double xe = lds_f64(sc + (p ? xro[i] : xlo[i]));  // the one x halo value needed
#pragma unroll
                    for (int jp = 0; jp < CPL / 2; ++jp) {
                        const int j0 = 2 * jp;
                        const uint32_t jb = 8u * (uint32_t)(j0 + p);
                        const double w_ = p ? uc[i][j0] : (jp == 0 ? xe : uc[i][j0 - 1]);
                        const double e_ = p ? (jp == CPL / 2 - 1 ? xe : uc[i][j0 + 2]) : uc[i][j0 + 1];
                        const double ym = i > 0 ? (p ? uc[i - 1][j0 + 1] : uc[i - 1][j0])
                                                : lds_f64(sc + roff[0] - ystep + jb);
                        const double yp = i < RPW - 1 ? (p ? uc[i + 1][j0 + 1] : uc[i + 1][j0])
                                                      : lds_f64(sc + ypo + jb);
                        const double zm = p ? um[i][j0 + 1] : um[i][j0];
                        const double zp = p ? un[i][j0 + 1] : un[i][j0];
                        const double rh = lds_f64(sc + rof[i] + jb);
                        double sum = rn_add(rn_add(rn_add(rn_add(rn_add(w_, e_), ym), yp), zm), zp);
                        const double upd = __ddiv_rn(rn_add(sum, rn_mul(h2, rh)), 6.0);
                        out[i][j0] = p ? uc[i][j0] : upd;
                        out[i][j0 + 1] = p ? upd : uc[i][j0 + 1];
                    }
                }
            }
            release(gc);
            auto st_cells = [&](double *d, int i) {
#pragma unroll
                for (int j = 0; j < CPL; j += (CPL >= 2 ? 2 : 1)) {
                    if constexpr (CPL >= 2)
                        *reinterpret_cast<double2 *>(d + j) = make_double2(out[i][j], out[i][j + 1]);
                    else
                        d[j] = out[i][j];
                }
            };
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                if (!on[i]) continue;
                st_cells(orow[i] + koff, i);
                if (i == ylo_i) st_cells(ylo + koff, i);
                if (i == yhi_i) st_cells(yhi + koff, i);
            }
            if (kk == kz_lo || kk == kz_hi) {
                const int64_t zd = kk == kz_lo ? zoff_lo : zoff_hi;
#pragma unroll
                for (int i = 0; i < RPW; ++i)
                    if (on[i]) st_cells(orow[i] + koff + zd, i);
            }
            if (xhp) {
#pragma unroll
                for (int i = 0; i < RPW; ++i)
                    if (on[i]) xhp[xk + i] = x_right ? out[i][CPL - 1] : out[i][0];
            }
            xk += xstep;
            koff += pstep;
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    um[i][j] = out[i][j];  // the plane as it is now (z-1 of the next plane)
                    uc[i][j] = un[i][j];
                }
        }
        release(g + nk + 1);
        g += nk + 2;
    }
}

}  // namespace

namespace {

template <int CPL, int NWARP, int RPW, bool PACKED, bool SCATTER, bool REV, bool NBRH, bool GW, bool HW = false,
          bool FILL = false>
int launch_march_one(const CUtensorMap &map, const CUtensorMap &xmap, const CUtensorMap &rmap, const MarchArgs &a,
                     int nctas, int ncomp, size_t smem, cudaStream_t s) {
    auto kern = march_kernel<CPL, NWARP, RPW, PACKED, SCATTER, REV, NBRH, GW, HW, FILL>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute(march)");
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nctas, ncomp);
    cfg.blockDim = dim3((NWARP + 1 + FILL) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, map, xmap, rmap, a);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "march launch");
    return TM_OK;
}

// TM_HALFWARP=0: boxes 18..32 wide keep one cell per lane (A/B measurements)
bool halfwarp_enabled() {
    static const bool on = [] {
        const char *e = getenv("TM_HALFWARP");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <bool PACKED, bool SCATTER, bool REV, bool NBRH = false, bool GW = false, bool FILL = false>
int launch_march(const CUtensorMap &map, const CUtensorMap &xmap, const CUtensorMap &rmap, const MarchArgs &a, int cpl,
                 int rows, int max_nx, int nctas, int ncomp, size_t smem, cudaStream_t s) {
    if (cpl == 1 && max_nx > 16 && rows <= 32 && halfwarp_enabled()) {  // half-warp row groups, 2 cells per lane
        if (rows <= 16)
            return launch_march_one<2, 4, 2, PACKED, SCATTER, REV, NBRH, GW, true, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
        return launch_march_one<2, 8, 2, PACKED, SCATTER, REV, NBRH, GW, true, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
    }
    // rows per CTA: 8 -> 4x2, 16 -> 8x2, 32 -> 16x2, 64 -> 16x4
    if (cpl == 2) {
        if (rows <= 8) return launch_march_one<2, 4, 2, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
        if (rows <= 14) return launch_march_one<2, 7, 2, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
        if (rows <= 16) return launch_march_one<2, 8, 2, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
        if (rows <= 32) return launch_march_one<2, 16, 2, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
        return launch_march_one<2, 16, 4, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
    }
    if (cpl == 4) {  // 4 cells per lane already give ILP: one or two rows per warp
        if (rows <= 8) return launch_march_one<4, 8, 1, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
        if (rows <= 16) return launch_march_one<4, 16, 1, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
        return launch_march_one<4, 16, 2, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
    }
    if (rows <= 8) return launch_march_one<1, 4, 2, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
    if (rows <= 16) return launch_march_one<1, 8, 2, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
    if (rows <= 32) return launch_march_one<1, 8, 4, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
    return launch_march_one<1, 16, 4, PACKED, SCATTER, REV, NBRH, GW, false, FILL>(map, xmap, rmap, a, nctas, ncomp, smem, s);
}


template <int CPL, int NWARP, int RPW>
int launch_gsrb_one(const CUtensorMap &map, const CUtensorMap &xmap, const CUtensorMap &rmap, const GsrbArgs &a,
                    int nctas, size_t smem, cudaStream_t s) {
    auto kern = gsrb_march_kernel<CPL, NWARP, RPW>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute(gsrb march)");
        configured = true;
    }
    kern<<<nctas, (NWARP + 1) * 32, smem, s>>>(map, xmap, rmap, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "gsrb march launch");
    return TM_OK;
}

int launch_gsrb(const CUtensorMap &map, const CUtensorMap &xmap, const CUtensorMap &rmap, const GsrbArgs &a, int cpl,
                int rows, int nctas, size_t smem, cudaStream_t s) {
    if (cpl == 2) {
        if (rows <= 8) return launch_gsrb_one<2, 4, 2>(map, xmap, rmap, a, nctas, smem, s);
        if (rows <= 16) return launch_gsrb_one<2, 8, 2>(map, xmap, rmap, a, nctas, smem, s);
        if (rows <= 32) return launch_gsrb_one<2, 8, 4>(map, xmap, rmap, a, nctas, smem, s);
        return launch_gsrb_one<2, 16, 4>(map, xmap, rmap, a, nctas, smem, s);
    }
    if (cpl == 4) {
        if (rows <= 8) return launch_gsrb_one<4, 8, 1>(map, xmap, rmap, a, nctas, smem, s);
        if (rows <= 16) return launch_gsrb_one<4, 16, 1>(map, xmap, rmap, a, nctas, smem, s);
        return launch_gsrb_one<4, 16, 2>(map, xmap, rmap, a, nctas, smem, s);
    }
    if (rows <= 8) return launch_gsrb_one<1, 4, 2>(map, xmap, rmap, a, nctas, smem, s);
    if (rows <= 16) return launch_gsrb_one<1, 8, 2>(map, xmap, rmap, a, nctas, smem, s);
    if (rows <= 32) return launch_gsrb_one<1, 8, 4>(map, xmap, rmap, a, nctas, smem, s);
    return launch_gsrb_one<1, 16, 4>(map, xmap, rmap, a, nctas, smem, s);
}

int encode_xh_map(CUtensorMap *map, const tm_layout &L, const double *xh, int box_y) {
    // packed x halo: dims (nyv, 2, nzv, nslots*ncomp), box (box_y, 2, 1, 1)
    tm_layout X{};
    X.nslots = L.nslots;
    X.ncomp = L.ncomp;
    X.nghost = 0;
    X.pitch = L.ny - 2 * L.nghost;  // nyv doubles per "row"
    X.ny = 2;
    X.nz = L.nz - 2 * L.nghost;
    X.xoff = 0;
    return tmk::encode_plane_map(map, X, xh, box_y, 2);
}

}  // namespace

extern "C" {

int tm_march_plan_create(const tm_block *cols, int64_t ncols, int32_t nctas, tm_march_plan **out) {
    using namespace tmk;
    if (!out) return fail(TM_ERR_INVALID, "tm_march_plan_create: null out");
    *out = nullptr;
    if (ncols < 0 || (ncols > 0 && !cols) || nctas < 1)
        return fail(TM_ERR_INVALID, "tm_march_plan_create: bad arguments");
    int64_t total = 0;
    int mx = 1, my = 1;
    bool even = true;
    for (int64_t c = 0; c < ncols; ++c) {
        const tm_block &k = cols[c];
        if (k.nx < 1 || k.ny < 1 || k.nz < 1 || k.x0 < 2 || k.y0 < 1 || k.z0 < 1)
            return fail(TM_ERR_INVALID, "tm_march_plan_create: malformed column " + std::to_string(c));
        total += k.nz;
        mx = std::max(mx, k.nx);
        my = std::max(my, k.ny);
        even = even && (k.x0 % 2 == 0) && (k.nx % 2 == 0);
    }
    if (mx > 128 || my > 64 || (mx > 64 && my > 32))
        return fail(TM_ERR_INVALID, "tm_march_plan_create: column exceeds 64 x 64 / 128 x 32");
    // equal contiguous shares of the column planes (reference partition rule, iterator.py:93-103)
    std::vector<Segment> segs;
    std::vector<int32_t> begin(nctas + 1, 0);
    int64_t col = 0, k = 0;
    for (int32_t i = 0; i < nctas; ++i) {
        begin[i] = (int32_t)segs.size();
        const int64_t q = total / nctas, r = total % nctas;
        int64_t left = q + (i < r ? 1 : 0);
        while (left > 0 && col < ncols) {
            const int64_t take = std::min<int64_t>(left, cols[col].nz - k);
            segs.push_back(Segment{(int32_t)col, (int32_t)k, (int32_t)(k + take), 0});
            k += take;
            left -= take;
            if (k == cols[col].nz) {
                ++col;
                k = 0;
            }
        }
    }
    begin[nctas] = (int32_t)segs.size();
    tm_march_plan *p = new tm_march_plan();
    p->ncols = ncols;
    p->nsegs = (int64_t)segs.size();
    p->nctas = nctas;
    p->max_nx = mx;
    p->max_ny = my;
    p->even = even;
    p->x0_common = ncols ? cols[0].x0 : -1;
    for (int64_t c = 0; c < ncols; ++c) {
        p->uniform_ny = p->uniform_ny && cols[c].ny == my;
        p->uniform_nx = p->uniform_nx && cols[c].nx == mx;
        p->ny_mult4 = p->ny_mult4 && cols[c].ny % 4 == 0;
        if (cols[c].x0 != p->x0_common) p->x0_common = -1;
    }
    cudaError_t e = cudaMalloc(&p->d_cols, sizeof(tm_block) * std::max<int64_t>(ncols, 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_segs, sizeof(Segment) * std::max<size_t>(segs.size(), 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_seg_begin, sizeof(int32_t) * (nctas + 1));
    if (e == cudaSuccess && ncols) e = cudaMemcpy(p->d_cols, cols, sizeof(tm_block) * ncols, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !segs.empty())
        e = cudaMemcpy(p->d_segs, segs.data(), sizeof(Segment) * segs.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_seg_begin, begin.data(), sizeof(int32_t) * (nctas + 1), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(p->d_cols);
        cudaFree(p->d_segs);
        cudaFree(p->d_seg_begin);
        delete p;
        return cuda_fail(e, "tm_march_plan_create");
    }
    *out = p;
    return TM_OK;
}

int tm_march_plan_destroy(tm_march_plan *p) {
    if (!p) return TM_OK;
    // tables may still be read by queued launches on any stream: drain before freeing
    cudaDeviceSynchronize();
    cudaFree(p->d_cols);
    cudaFree(p->d_segs);
    cudaFree(p->d_seg_begin);
    cudaFree(p->d_peer_maps);
    delete p;
    return TM_OK;
}

int tm_march_plan_reset_halos(tm_march_plan *p) {
    if (!p) return tmk::fail(TM_ERR_INVALID, "tm_march_plan_reset_halos: null plan");
    p->last_halo_mode = -1;
    p->last_xh_new = nullptr;
    return TM_OK;
}

}  // extern "C"

namespace {

int heat_march_impl(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew, int32_t ncomp_sweep,
                    double dxi0, double dxi1, double dxi2, double dtD, int32_t halo_mode, const double *xh_old,
                    double *xh_new, const int32_t *d_nbr, int32_t reverse, const int64_t *fill_cells, int64_t nfill,
                    void *stream, int32_t peer_set = -1) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, "tm_heat_march: null plan");
    int rc = check_layout(layout, "tm_heat_march");
    if (rc) return rc;
    const tm_layout &L = *layout;
    if (L.nghost < 1 || !uold || !unew || uold == unew)
        return fail(TM_ERR_INVALID, "tm_heat_march: needs nghost >= 1 and distinct old/new fields");
    if (ncomp_sweep < 1 || ncomp_sweep > L.ncomp) return fail(TM_ERR_INVALID, "tm_heat_march: bad ncomp");
    if (strides_of(L).comp >= ((int64_t)1 << 32))
        return fail(TM_ERR_INVALID, "tm_heat_march: one component of a slot must hold < 2^32 doubles");
    const bool nbr_mode = halo_mode == TM_HALO_FUSED_NBR || halo_mode == TM_HALO_FUSED_NBR_GHOSTS;
    const bool packed = halo_mode == TM_HALO_PACKED || halo_mode == TM_HALO_FUSED_SCATTER || nbr_mode;
    const bool scatter = halo_mode == TM_HALO_FUSED_SCATTER || nbr_mode || halo_mode == TM_HALO_GHOSTS_XH;
    switch (halo_mode) {
        case TM_HALO_GHOSTS:
            if (xh_old || xh_new || d_nbr || reverse)
                return fail(TM_ERR_INVALID, "tm_heat_march: TM_HALO_GHOSTS takes no halo buffers, table or reverse");
            break;
        case TM_HALO_PACKED:
            if (!xh_old || xh_new || d_nbr || reverse)
                return fail(TM_ERR_INVALID, "tm_heat_march: TM_HALO_PACKED needs xh_old only");
            break;
        case TM_HALO_GHOSTS_XH:
            if (xh_old || !xh_new || !d_nbr)
                return fail(TM_ERR_INVALID, "tm_heat_march: TM_HALO_GHOSTS_XH needs xh_new and d_nbr, no xh_old");
            break;
        case TM_HALO_FUSED_SCATTER:
        case TM_HALO_FUSED_NBR:
        case TM_HALO_FUSED_NBR_GHOSTS:
            if (!xh_old || !xh_new || !d_nbr || xh_old == xh_new)
                return fail(TM_ERR_INVALID, "tm_heat_march: fused modes need distinct xh_old / xh_new and d_nbr");
            if (halo_mode == TM_HALO_FUSED_NBR_GHOSTS && (reverse || L.nghost != 1 || L.xoff < 4))
                return fail(TM_ERR_INVALID, "tm_heat_march: TM_HALO_FUSED_NBR_GHOSTS is forward, nghost 1");
            break;
        default:
            return fail(TM_ERR_INVALID, "tm_heat_march: unknown halo_mode " + std::to_string(halo_mode));
    }
    if (p->ncols == 0) return TM_OK;
    if (!p->even) return fail(TM_ERR_INVALID, "tm_heat_march: columns must start on even x and have even width");
    const int cpl = p->max_nx <= 32 ? 1 : (p->max_nx <= 64 ? 2 : 4);
    if (cpl == 4 && (p->max_nx % 4)) return fail(TM_ERR_INVALID, "tm_heat_march: widths > 64 must be multiples of 4");
    if ((packed || scatter) && p->max_ny % 2)
        return fail(TM_ERR_INVALID, "tm_heat_march: packed x halos need even column heights");
    // neighbour-sourced y/z halos: the column rows and the two halo rows are separate TMA boxes,
    // each landing on a stage row that must be 128-B aligned (TMA destination)
    if (nbr_mode && !(p->uniform_ny && p->max_nx % 16 == 0))
        return fail(TM_ERR_INVALID, "tm_heat_march: TM_HALO_FUSED_NBR needs columns of one height and a width that "
                                    "is a multiple of 16");
    // A TM_HALO_FUSED_NBR step leaves the y/z face ghosts of unew unwritten; a following
    // TM_HALO_FUSED_SCATTER step would read them.  Refuse that hand-over (tm_march_plan_reset_halos
    // after a FillBoundary re-arms the plan).
    if (halo_mode == TM_HALO_FUSED_SCATTER && p->last_halo_mode == TM_HALO_FUSED_NBR && xh_old == p->last_xh_new)
        return fail(TM_ERR_INVALID, "tm_heat_march: TM_HALO_FUSED_SCATTER after a TM_HALO_FUSED_NBR step reads y/z "
                                    "ghosts that step did not write; FillBoundary + tm_march_plan_reset_halos first");
    MarchArgs a{};
    a.cols = p->d_cols;
    a.segs = p->d_segs;
    a.seg_begin = p->d_seg_begin;
    a.out = unew;
    a.L = L;
    a.c0 = dxi0;
    a.c1 = dxi1;
    a.c2 = dxi2;
    a.c3 = dtD;
    a.box_x = packed ? p->max_nx : p->max_nx + 4;
    a.box_y = p->max_ny + 2;
    a.nyv = L.ny - 2 * L.nghost;
    a.nzv = L.nz - 2 * L.nghost;
    a.xh_off = ((a.box_x * a.box_y + 15) / 16) * 16;
    const int stage = packed ? a.xh_off + ((2 * p->max_ny + 15) / 16) * 16 : a.xh_off;
    a.stage_elems = stage;
    a.xh_new = xh_new;
    a.nbr = d_nbr;
    a.gw = const_cast<double *>(uold);  // TM_HALO_FUSED_NBR_GHOSTS only: uold's face ghosts (documented)
    if (peer_set >= 0) {
        if (halo_mode != TM_HALO_FUSED_NBR)
            return fail(TM_ERR_INVALID, "tm_heat_march_peer: peer faces ride on TM_HALO_FUSED_NBR");
        if (peer_set >= TM_PEER_SETS || p->peer_n[peer_set] < 0)
            return fail(TM_ERR_INVALID, "tm_heat_march_peer: peer set " + std::to_string(peer_set) +
                                            " not encoded (tm_march_plan_set_peers)");
        if (p->peer_box_x != a.box_x || p->peer_box_y != p->max_ny)
            return fail(TM_ERR_INVALID, "tm_heat_march_peer: peer maps encoded for another column box");
        a.pmaps = p->d_peer_maps + (size_t)peer_set * TM_MAX_PEERS * 2;
    }
    const size_t smem = (size_t)kHeatStages * stage * sizeof(double) + 2 * kHeatStages * sizeof(uint64_t);
    if (smem > 220 * 1024) return fail(TM_ERR_INVALID, "tm_heat_march: column plane too large for shared memory");
    CUtensorMap map, xmap;
    rc = encode_plane_map(&map, L, uold, a.box_x, a.box_y);
    if (rc) return rc;
    if (packed) {
        rc = encode_xh_map(&xmap, L, xh_old, p->max_ny);
        if (rc) return rc;
    } else {
        xmap = map;
    }
    cudaStream_t s = as_stream(stream);
    if (scatter) {
        p->last_halo_mode = halo_mode;
        p->last_xh_new = xh_new;
    }
    if (halo_mode == TM_HALO_GHOSTS_XH)
        return launch_march<false, true, false>(map, xmap, map, a, cpl, p->max_ny, p->max_nx, p->nctas, ncomp_sweep, smem, s);
    switch (halo_mode) {
        case TM_HALO_GHOSTS:
            return launch_march<false, false, false>(map, xmap, map, a, cpl, p->max_ny, p->max_nx, p->nctas, ncomp_sweep, smem, s);
        case TM_HALO_PACKED:
            return launch_march<true, false, false>(map, xmap, map, a, cpl, p->max_ny, p->max_nx, p->nctas, ncomp_sweep, smem, s);
        case TM_HALO_FUSED_NBR_GHOSTS:
        case TM_HALO_FUSED_NBR: {
            CUtensorMap cmap, rmap;
            rc = encode_plane_map(&cmap, L, uold, a.box_x, p->max_ny);
            if (rc) return rc;
            rc = encode_plane_map(&rmap, L, uold, a.box_x, 1);
            if (rc) return rc;
            if (halo_mode == TM_HALO_FUSED_NBR_GHOSTS && fill_cells && nfill > 0) {
                a.fcells = fill_cells;
                a.nfcells = nfill;
                return launch_march<true, true, false, true, true, true>(cmap, xmap, rmap, a, cpl, p->max_ny,
                                                                         p->max_nx, p->nctas, ncomp_sweep, smem, s);
            }
            if (halo_mode == TM_HALO_FUSED_NBR_GHOSTS)
                return launch_march<true, true, false, true, true>(cmap, xmap, rmap, a, cpl, p->max_ny, p->max_nx, p->nctas,
                                                                   ncomp_sweep, smem, s);
            if (reverse)
                return launch_march<true, true, true, true>(cmap, xmap, rmap, a, cpl, p->max_ny, p->max_nx, p->nctas, ncomp_sweep,
                                                            smem, s);
            return launch_march<true, true, false, true>(cmap, xmap, rmap, a, cpl, p->max_ny, p->max_nx, p->nctas, ncomp_sweep,
                                                         smem, s);
        }
        default:
            if (reverse)
                return launch_march<true, true, true>(map, xmap, map, a, cpl, p->max_ny, p->max_nx, p->nctas, ncomp_sweep, smem, s);
            return launch_march<true, true, false>(map, xmap, map, a, cpl, p->max_ny, p->max_nx, p->nctas, ncomp_sweep, smem, s);
    }
}

}  // namespace

extern "C" {

int tm_heat_march(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew, int32_t ncomp_sweep,
                  double dxi0, double dxi1, double dxi2, double dtD, int32_t halo_mode, const double *xh_old,
                  double *xh_new, const int32_t *d_nbr, int32_t reverse, void *stream) {
    return heat_march_impl(p, layout, uold, unew, ncomp_sweep, dxi0, dxi1, dxi2, dtD, halo_mode, xh_old, xh_new,
                           d_nbr, reverse, nullptr, 0, stream);
}

int tm_march_plan_set_peers(tm_march_plan *p, int32_t set, const tm_layout *layout, int32_t npeers,
                            const double *const *peer_base, const int64_t *peer_nslots) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, "tm_march_plan_set_peers: null plan");
    int rc = check_layout(layout, "tm_march_plan_set_peers");
    if (rc) return rc;
    if (set < 0 || set >= TM_PEER_SETS) return fail(TM_ERR_INVALID, "tm_march_plan_set_peers: bad set");
    if (npeers < 0 || npeers > TM_MAX_PEERS || (npeers && (!peer_base || !peer_nslots)))
        return fail(TM_ERR_INVALID, "tm_march_plan_set_peers: 0..TM_MAX_PEERS peers with bases and slot counts");
    if (p->ncols && !(p->uniform_ny && p->max_nx % 16 == 0))
        return fail(TM_ERR_INVALID, "tm_march_plan_set_peers: peer faces need the neighbour-halo march "
                                    "(columns of one height, width a multiple of 16)");
    if (!p->d_peer_maps) {
        cudaError_t e = cudaMalloc(&p->d_peer_maps, sizeof(CUtensorMap) * TM_PEER_SETS * TM_MAX_PEERS * 2);
        if (e != cudaSuccess) return cuda_fail(e, "tm_march_plan_set_peers: cudaMalloc");
    }
    // the column box of the fused (packed) march: max_nx x max_ny rows, and a one-row box
    const int bx = p->max_nx, by = p->max_ny;
    CUtensorMap maps[TM_MAX_PEERS * 2];
    memset(maps, 0, sizeof(maps));
    for (int i = 0; i < npeers; ++i) {
        if (!peer_base[i] || peer_nslots[i] < 1)
            return fail(TM_ERR_INVALID, "tm_march_plan_set_peers: peer " + std::to_string(i) + " has no storage");
        tm_layout P = *layout;
        P.nslots = peer_nslots[i];
        if (p->ncols) {
            rc = encode_plane_map(&maps[2 * i], P, peer_base[i], bx, by);
            if (rc) return rc;
            rc = encode_plane_map(&maps[2 * i + 1], P, peer_base[i], bx, 1);
            if (rc) return rc;
        }
    }
    // synchronous upload: setup time, outside any capture; queued launches of this plan may
    // still read the set's previous maps, so drain first
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "tm_march_plan_set_peers: synchronize");
    e = cudaMemcpy(p->d_peer_maps + (size_t)set * TM_MAX_PEERS * 2, maps, sizeof(maps), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "tm_march_plan_set_peers: cudaMemcpy");
    p->peer_n[set] = npeers;
    p->peer_box_x = bx;
    p->peer_box_y = by;
    return TM_OK;
}

int tm_heat_march_peer(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                       int32_t ncomp_sweep, double dxi0, double dxi1, double dxi2, double dtD, const double *xh_old,
                       double *xh_new, const int32_t *d_nbr, int32_t set, int32_t reverse, void *stream) {
    if (set < 0) return tmk::fail(TM_ERR_INVALID, "tm_heat_march_peer: bad peer set");
    return heat_march_impl(p, layout, uold, unew, ncomp_sweep, dxi0, dxi1, dxi2, dtD, TM_HALO_FUSED_NBR, xh_old,
                           xh_new, d_nbr, reverse, nullptr, 0, stream, set);
}

int tm_heat_march_fill(tm_march_plan *p, const tm_layout *layout, const double *uold, double *unew,
                       int32_t ncomp_sweep, double dxi0, double dxi1, double dxi2, double dtD, const double *xh_old,
                       double *xh_new, const int32_t *d_nbr, const int64_t *d_fill_cells, int64_t nfill_cells,
                       void *stream) {
    if (nfill_cells < 0 || (nfill_cells > 0 && !d_fill_cells) ||
        (reinterpret_cast<uintptr_t>(d_fill_cells) & 15) != 0)
        return tmk::fail(TM_ERR_INVALID, "tm_heat_march_fill: bad cell list (16-B aligned int64 pairs)");
    return heat_march_impl(p, layout, uold, unew, ncomp_sweep, dxi0, dxi1, dxi2, dtD, TM_HALO_FUSED_NBR_GHOSTS, xh_old,
                           xh_new, d_nbr, 0, d_fill_cells, nfill_cells, stream);
}

int tm_gsrb_march(tm_march_plan *p, const tm_layout *phi_layout, double *phi, const tm_layout *rhs_layout,
                  const double *rhs, int32_t color, double h2, double *xh, const int32_t *d_nbr, void *stream) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, "tm_gsrb_march: null plan");
    int rc = check_layout(phi_layout, "tm_gsrb_march");
    if (rc) return rc;
    rc = check_layout(rhs_layout, "tm_gsrb_march(rhs)");
    if (rc) return rc;
    const tm_layout &L = *phi_layout;
    if (L.nghost < 1 || L.ncomp != 1 || rhs_layout->ncomp != 1 || !phi || !rhs || !xh || !d_nbr ||
        (color != 0 && color != 1))
        return fail(TM_ERR_INVALID, "tm_gsrb_march: bad arguments");
    if (p->ncols == 0) return TM_OK;
    if (!p->even || p->max_ny % 2) return fail(TM_ERR_INVALID, "tm_gsrb_march: columns must be even-sized");
    if (strides_of(L).comp >= ((int64_t)1 << 32))
        return fail(TM_ERR_INVALID, "tm_gsrb_march: one slot must hold < 2^32 doubles");
    GsrbArgs ga{};
    MarchArgs &a = ga.m;
    a.cols = p->d_cols;
    a.segs = p->d_segs;
    a.seg_begin = p->d_seg_begin;
    a.out = phi;
    a.L = L;
    a.box_x = p->max_nx;
    a.box_y = p->max_ny + 2;
    a.nyv = L.ny - 2 * L.nghost;
    a.nzv = L.nz - 2 * L.nghost;
    a.xh_off = ((a.box_x * a.box_y + 15) / 16) * 16;
    ga.rhs_off = a.xh_off + ((2 * p->max_ny + 15) / 16) * 16;
    a.stage_elems = ga.rhs_off + ((p->max_nx * p->max_ny + 15) / 16) * 16;
    a.xh_new = xh;
    a.nbr = d_nbr;
    ga.R = *rhs_layout;
    ga.color = color;
    ga.h2 = h2;
    const size_t smem = (size_t)kGsrbStages * a.stage_elems * sizeof(double) + 2 * kGsrbStages * sizeof(uint64_t);
    if (smem > 220 * 1024) return fail(TM_ERR_INVALID, "tm_gsrb_march: column plane too large for shared memory");
    CUtensorMap map, xmap, rmap;
    rc = encode_plane_map(&map, L, phi, a.box_x, a.box_y);
    if (rc) return rc;
    rc = encode_xh_map(&xmap, L, xh, p->max_ny);
    if (rc) return rc;
    rc = encode_plane_map(&rmap, *rhs_layout, rhs, p->max_nx, p->max_ny);
    if (rc) return rc;
    const int cpl = p->max_nx <= 32 ? 1 : (p->max_nx <= 64 ? 2 : 4);
    if (cpl == 4 && (p->max_nx % 4)) return fail(TM_ERR_INVALID, "tm_gsrb_march: widths > 64 must be multiples of 4");
    return launch_gsrb(map, xmap, rmap, ga, cpl, p->max_ny, p->nctas, smem, as_stream(stream));
}

}  // extern "C"
