// Red-black Gauss-Seidel on colour-split storage ("caps GSRB
// at about 50 % of this roofline unless the layout ... changes").
//
// During a solve each colour of phi lives in its own array, a row holding only
// that colour's cells: entry i of row (y, z) is the cell x = 2i + o_c(y, z),
// o_c = (c + x_lo + y + z) & 1 (global parity of the box origin), i in
// [-1, nx/2] so each row also carries its one x-ghost cell of that colour.
// Layout per colour: [slot][z+1][y+1][i+2], rows nx/2 + 4 doubles wide; the
// rhs is split once per solve into [slot][z][y][i].  A colour-c pass reads
// only the other colour's array and colour c's rhs and writes colour c's
// array: 8 + 8 + 8 bytes per UPDATED cell (half the cells) instead of
// 24 bytes per cell, and no pass ever reads what it writes.
//
// Per updated cell, with w/e the x neighbours, s/n the y neighbours and b/t
// the z neighbours (all the other colour):
//   w = O[i-1+o], e = O[i+o] (same row), s/n = O[i] of rows y-1 / y+1,
//   b/t = O[i] of planes z-1 / z+1
//   phi = (((((w + e) + s) + n) + b) + t + h2*rhs) / 6
// -- the builder-owned form of tm_gsrb_color (oracle/tm_oracle.c), bit for bit.
// The epilogue scatters the box's new boundary values of colour c into the
// face neighbours' ghost entries of the same colour array (the fused
// FillBoundary of BASELINE config 4).  Requires uniform boxes, nx % 4 == 0,
// even periodic extents (so a periodic image has the same colouring).
#include <string>

#include "tm_march_plan.cuh"

namespace {

using tmk::Segment;

constexpr int kSStages = 8;  // 4: 51.1 us per C4 pass, 8: 50.5 (16-row columns) / 48.9 (32 rows)

// Entry e of a colour row sits at index e + kE0 of a row of wp = nx/2 + 8 doubles
// (320 B for 64-wide boxes): every row's valid entries start on a 32-B sector
// boundary, so a pass writes whole sectors (no partial-sector write-back);
// TMA loads rows from entry -2 (index 2, 16-B aligned), nx/2 + 4 doubles wide.
constexpr int kE0 = 4;

struct ColourLayout {
    int32_t nslots, nx, ny, nz;  // valid extents of every box
    int32_t wp;                  // doubles per colour row: nx/2 + 8
    int64_t row, plane, slot;    // strides of a colour array
    int64_t rrow, rplane, rslot; // strides of a colour rhs array (nx/2 per row, valid rows only)
};

__host__ __device__ inline ColourLayout colour_layout(int nslots, int nx, int ny, int nz) {
    ColourLayout C;
    C.nslots = nslots;
    C.nx = nx;
    C.ny = ny;
    C.nz = nz;
    // 320-B rows for 64-wide boxes: row pitches of 304 / 336 / 352 / 384 / 448 B measured 54.0 /
    // 60.8 / 53.7 / 61.2 / 64.4 us per C4 pass against 48.9 (r02); plane padding: no effect
    C.wp = nx / 2 + 8;
    C.row = C.wp;
    C.plane = C.row * (ny + 2);
    C.slot = C.plane * (nz + 2);
    C.rrow = nx / 2;
    C.rplane = C.rrow * ny;
    C.rslot = C.rplane * nz;
    return C;
}

// phi (valid + one ghost layer) -> both colour arrays; rhs -> both colour rhs arrays.
// One warp per row (slot, z, y): lane l loads the cell pair x = 2l, 2l+1 with one 16-B load
// (rows start 128-B aligned), which holds entry l of both colours -- colour c's entry sits at
// offset o_c = (c + parity + y + z) & 1 of the pair -- and stores them with two coalesced
// 8-B stores.  The two x-ghost entries (x = -1 and x = nx) come from lanes 0 and 31.
// (r01's thread-per-entry gather: 242 us per C4 solve for split, 114 for merge + fill.)
__global__ void split_kernel(tm_layout L, const double *__restrict__ phi, ColourLayout C, const int32_t *parity,
                             double *__restrict__ c0, double *__restrict__ c1, tm_layout R,
                             const double *__restrict__ rhs, double *__restrict__ r0, double *__restrict__ r1) {
    // kB rows per warp and trip, their loads issued together (one row in flight per warp left
    // the kernel latency-bound: 187 us per C4 split); 32-bit row indices (host-checked)
    constexpr int kB = 4;
    const int nh = C.nx / 2;
    const int lane = threadIdx.x & 31;
    const int rows = C.nslots * (C.nz + 2) * (C.ny + 2);
    const int wstride = gridDim.x * (blockDim.x >> 5) * kB;
    const tmk::Strides s = tmk::strides_of(L);
    const tmk::Strides rs = tmk::strides_of(R);
    for (int t0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kB; t0 < rows; t0 += wstride) {
        for (int e = lane; e < nh; e += 32) {
            double2 v[kB], rv[kB];
            int o0[kB];
            bool vr[kB];
            int64_t dro[kB], rro[kB];
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int t = min(t0 + b, rows - 1);
                const int yy = t % (C.ny + 2), zs = t / (C.ny + 2);
                const int zz = zs % (C.nz + 2), slot = zs / (C.nz + 2);
                const int y = yy - 1, z = zz - 1;
                o0[b] = (parity[slot] + y + z) & 1;  // x offset of colour 0's entries in this row
                dro[b] = slot * C.slot + (int64_t)zz * C.plane + (int64_t)yy * C.row + kE0;
                v[b] = *reinterpret_cast<const double2 *>(phi + slot * s.slot + (int64_t)(z + L.nghost) * s.plane +
                                                          (int64_t)(y + L.nghost) * s.row + L.xoff + 2 * e);
                vr[b] = rhs && y >= 0 && y < C.ny && z >= 0 && z < C.nz && t0 + b < rows;
                rro[b] = slot * C.rslot + (int64_t)z * C.rplane + (int64_t)y * C.rrow;
                if (vr[b])
                    rv[b] = *reinterpret_cast<const double2 *>(rhs + slot * rs.slot + (int64_t)(z + R.nghost) * rs.plane +
                                                               (int64_t)(y + R.nghost) * rs.row + R.xoff + 2 * e);
            }
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                if (t0 + b >= rows) continue;
                c0[dro[b] + e] = o0[b] ? v[b].y : v[b].x;
                c1[dro[b] + e] = o0[b] ? v[b].x : v[b].y;
                if (vr[b]) {
                    r0[rro[b] + e] = o0[b] ? rv[b].y : rv[b].x;
                    r1[rro[b] + e] = o0[b] ? rv[b].x : rv[b].y;
                }
            }
        }
        // ghost entries: entry -1 of the colour at offset 1 is x = -1, entry nh of the colour at
        // offset 0 is x = nx
        if (lane < 2 * kB) {
            const int t = t0 + (lane >> 1);
            if (t < rows) {
                const int yy = t % (C.ny + 2), zs = t / (C.ny + 2);
                const int zz = zs % (C.nz + 2), slot = zs / (C.nz + 2);
                const int y = yy - 1, z = zz - 1;
                const int o0 = (parity[slot] + y + z) & 1;
                const double *prow = phi + slot * s.slot + (int64_t)(z + L.nghost) * s.plane +
                                     (int64_t)(y + L.nghost) * s.row + L.xoff;
                const int64_t ro = slot * C.slot + (int64_t)zz * C.plane + (int64_t)yy * C.row + kE0;
                if ((lane & 1) == 0)
                    (o0 ? c0 : c1)[ro - 1] = prow[-1];
                else
                    (o0 ? c1 : c0)[ro + nh] = prow[C.nx];
            }
        }
    }
}

// both colour arrays -> phi valid cells (one warp per kB rows, one 16-B store per cell pair)
__global__ void merge_kernel(tm_layout L, double *__restrict__ phi, ColourLayout C, const int32_t *parity,
                             const double *__restrict__ c0, const double *__restrict__ c1) {
    constexpr int kB = 4;
    const int nh = C.nx / 2;
    const int lane = threadIdx.x & 31;
    const int rows = C.nslots * C.nz * C.ny;
    const int wstride = gridDim.x * (blockDim.x >> 5) * kB;
    const tmk::Strides s = tmk::strides_of(L);
    for (int t0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kB; t0 < rows; t0 += wstride) {
        for (int e = lane; e < nh; e += 32) {
            double a0[kB], a1[kB];
            double *dst[kB];
            int o0[kB];
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int t = min(t0 + b, rows - 1);
                const int y = t % C.ny, zs = t / C.ny;
                const int z = zs % C.nz, slot = zs / C.nz;
                o0[b] = (parity[slot] + y + z) & 1;
                const int64_t ro = slot * C.slot + (int64_t)(z + 1) * C.plane + (int64_t)(y + 1) * C.row + kE0 + e;
                a0[b] = c0[ro];
                a1[b] = c1[ro];
                dst[b] = phi + slot * s.slot + (int64_t)(z + L.nghost) * s.plane + (int64_t)(y + L.nghost) * s.row +
                         L.xoff + 2 * e;
            }
#pragma unroll
            for (int b = 0; b < kB; ++b)
                if (t0 + b < rows)
                    *reinterpret_cast<double2 *>(dst[b]) =
                        o0[b] ? make_double2(a1[b], a0[b]) : make_double2(a0[b], a1[b]);
        }
    }
}

struct SplitArgs {
    const tm_block *cols;
    const Segment *segs;
    const int32_t *seg_begin;
    ColourLayout C;
    double *out;           // colour-c array (written)
    const int32_t *nbr;    // 6 face neighbours per slot (-x,+x,-y,+y,-z,+z)
    int32_t color;
    double h2;
    int32_t box_y, stage_elems, rhs_off;  // other-colour box rows (R+2), stage stride, rhs slice offset
};

template <int CPL, int NWARP, int RPW>
__global__ void __launch_bounds__((NWARP + 1) * 32, NWARP <= 8 ? 2 : 1)
    split_pass_kernel(const __grid_constant__ CUtensorMap omap, const __grid_constant__ CUtensorMap rmap, SplitArgs a) {
    using namespace tmk;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kSStages * a.stage_elems * sizeof(double));
    uint64_t *empty = bars + kSStages;
    const ColourLayout &C = a.C;
    const int s_begin = a.seg_begin[blockIdx.x], s_end = a.seg_begin[blockIdx.x + 1];
    if (s_begin >= s_end) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nh = C.nx / 2, wp = nh + 4;  // wp here: the staged row width (entries -2 .. nh+1)
    const int R = a.box_y - 2;
    const uint32_t tx_bytes = (uint32_t)((wp * a.box_y + nh * R) * (int)sizeof(double));

    if (tid == 0) {
        prefetch_tensormap(&omap);
        prefetch_tensormap(&rmap);
#pragma unroll
        for (int s = 0; s < kSStages; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&empty[s], NWARP);
        }
        fence_mbar_init();
    }
    grid_dep_launch();  // the next pass's CTAs may take SM slots as ours retire
    __syncthreads();
    grid_dep_wait();  // previous pass complete: it wrote the colour we read (and read the one we write)

    if (warp == NWARP) {  // ---------------- producer warp ----------------
        if (lane == 0) {
            int p = 0;
            for (int s = s_begin; s < s_end; ++s) {
                const Segment sg = a.segs[s];
                const tm_block c = a.cols[sg.col];
                const int yv = c.y0 - 1, zv0 = c.z0 - 1;  // valid y / z of the column's first row / plane
                const int n = sg.k1 - sg.k0 + 2;
                for (int q = 0; q < n; ++q, ++p) {
                    const int st_i = p % kSStages;
                    if (p >= kSStages) mbar_wait(&empty[st_i], ((p / kSStages) - 1) & 1);
                    double *stage = stages + st_i * a.stage_elems;
                    const int zv = zv0 + sg.k0 - 1 + q;  // valid z of this plane (-1 .. nz)
                    mbar_arrive_expect_tx(&bars[st_i], tx_bytes);
                    // other colour: rows yv-1 .. yv+R (array rows yv .. yv+R+1), plane zv (array zv+1)
                    tma_load_plane(stage, &omap, &bars[st_i], kE0 - 2, yv, zv + 1, c.slot);
                    // rhs of this colour (out-of-range halo planes read as zeros, never used)
                    tma_load_plane(stage + a.rhs_off, &rmap, &bars[st_i], 0, yv, zv, c.slot);
                }
            }
        }
        return;
    }

    // ---------------- consumer warps ----------------
    const uint32_t sbase = smem_u32(stages);
    const uint32_t bfull = smem_u32(bars), bempty = smem_u32(empty);
    const uint32_t sbytes = (uint32_t)a.stage_elems * 8u;
    auto saddr = [&](uint32_t q) { return sbase + (q & (kSStages - 1)) * sbytes; };
    auto wait_plane = [&](uint32_t q) { mbar_wait_u32(bfull + (q & (kSStages - 1)) * 8u, (q / kSStages) & 1u); };
    auto release = [&](uint32_t q) {
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bempty + (q & (kSStages - 1)) * 8u);
    };
    const double h2 = a.h2;
    const uint32_t ystep = (uint32_t)wp * 8u;
    // Hot-loop bookkeeping: per-segment row pointers and scatter targets, one running 32-bit
    // plane offset and a parity bit that flips per plane (r01 recomputed 64-bit addresses and
    // every scatter condition per cell).  Neither this, an 8-deep ring nor an early stage
    // release moves the pass much (50.8 / 50.5 / 52.1 us, r02): it streams at ~4.7 TB/s.
    const uint32_t cplane = (uint32_t)C.plane;  // host-checked < 2^31
    uint32_t g = 0;
    for (int s = s_begin; s < s_end; ++s) {
        const Segment sg = a.segs[s];
        const tm_block c = a.cols[sg.col];
        const int nk = sg.k1 - sg.k0;
        const int yv0 = c.y0 - 1, zv0 = c.z0 - 1 + sg.k0;  // valid y of row 0, valid z of the first plane
        const int32_t *nbp = a.nbr + 6 * c.slot;
        const bool lane_on = lane * CPL < nh;
        const int ii = min(lane * CPL, nh - CPL);  // lane's first entry
        uint32_t so[RPW], ro[RPW];  // stage byte offsets: other colour at (row, entry ii), rhs
        double *orow[RPW];          // colour-c cells of the row at the segment's first plane
        double *ysc[RPW];           // the -y / +y neighbour's ghost row entry, or null
        bool on[RPW];
        int o0[RPW];                // entry -> x offset of the colour at plane k0 (flips per plane)
        double *const sbase_out = a.out + (int64_t)c.slot * C.slot + (int64_t)(zv0 + 1) * C.plane + (ii + kE0);
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int r = warp * RPW + i;
            on[i] = lane_on && r < c.ny;
            const int rc = min(r, R - 1);
            so[i] = (uint32_t)((rc + 1) * wp + ii + 2) * 8u;
            ro[i] = (uint32_t)(a.rhs_off + rc * nh + ii) * 8u;
            orow[i] = sbase_out + (int64_t)(yv0 + r + 1) * C.row;
            o0[i] = (a.color + c.parity + r + sg.k0) & 1;
            const int yv = yv0 + r;
            ysc[i] = nullptr;
            if (on[i] && yv == 0 && nbp[2] >= 0)  // row 0 -> the -y neighbour's row ny
                ysc[i] = orow[i] + (int64_t)(nbp[2] - c.slot) * C.slot + (int64_t)C.ny * C.row;
            else if (on[i] && yv == C.ny - 1 && nbp[3] >= 0)  // row ny-1 -> the +y neighbour's row -1
                ysc[i] = orow[i] + (int64_t)(nbp[3] - c.slot) * C.slot - (int64_t)C.ny * C.row;
        }
        // x faces: entry 0 at offset 0 is x = 0 (-> the -x neighbour's entry nh); entry nh-1 at
        // offset 1 is x = nx-1 (-> the +x neighbour's entry -1)
        const bool xlo = lane_on && ii == 0 && nbp[0] >= 0;
        const bool xhi = lane_on && ii + CPL == nh && nbp[1] >= 0;
        const int64_t dxlo = (int64_t)(nbp[0] - c.slot) * C.slot + nh;
        const int64_t dxhi = (int64_t)(nbp[1] - c.slot) * C.slot - nh;
        // z faces: plane 0 -> the -z neighbour's plane nz, plane nz-1 -> the +z neighbour's plane -1
        const int kzlo = (nbp[4] >= 0 && zv0 <= 0 && 0 < zv0 + nk) ? -zv0 : -1;
        const int kzhi = (nbp[5] >= 0 && zv0 <= C.nz - 1 && C.nz - 1 < zv0 + nk) ? C.nz - 1 - zv0 : -1;
        const int64_t dzlo = (int64_t)(nbp[4] - c.slot) * C.slot + (int64_t)C.nz * C.plane;
        const int64_t dzhi = (int64_t)(nbp[5] - c.slot) * C.slot - (int64_t)C.nz * C.plane;
        // z march state per cell: the other colour's value below (carried)
        double ob[RPW][CPL];
        wait_plane(g);
        wait_plane(g + 1);  // the first centre plane
        {
            const uint32_t s0 = saddr(g);
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; ++j) ob[i][j] = lds_f64(s0 + so[i] + 8u * j);
        }
        release(g);
        uint32_t kofs = 0;  // kk * C.plane
        for (int kk = 0; kk < nk; ++kk) {
            const uint32_t gc = g + 1 + (uint32_t)kk;
            wait_plane(gc + 1);
            const uint32_t sc = saddr(gc), sn = saddr(gc + 1);
            double out[RPW][CPL];
            int oo[RPW];
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                oo[i] = o0[i] ^ (kk & 1);
                const uint32_t ox = 8u * (uint32_t)oo[i];
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    const uint32_t p = sc + so[i] + 8u * j;
                    const double w = lds_f64(p - 8u + ox), e = lds_f64(p + ox);
                    const double sv = lds_f64(p - ystep), nv = lds_f64(p + ystep);
                    const double t = lds_f64(sn + so[i] + 8u * j);
                    const double rh = lds_f64(sc + ro[i] + 8u * j);
                    double sum = rn_add(rn_add(rn_add(rn_add(rn_add(w, e), sv), nv), ob[i][j]), t);
                    out[i][j] = __ddiv_rn(rn_add(sum, rn_mul(h2, rh)), 6.0);
                    ob[i][j] = lds_f64(p);  // this plane's other-colour value: "below" for the next plane
                }
            }
            release(gc);
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
                if (!on[i]) continue;
                double *d = orow[i] + kofs;
#pragma unroll
                for (int j = 0; j < CPL; ++j) d[j] = out[i][j];
                // fused FillBoundary of this colour: the face neighbours' ghost entries
                if (ysc[i]) {
#pragma unroll
                    for (int j = 0; j < CPL; ++j) ysc[i][kofs + j] = out[i][j];
                }
                if (kk == kzlo) {
#pragma unroll
                    for (int j = 0; j < CPL; ++j) d[dzlo + j] = out[i][j];
                }
                if (kk == kzhi) {
#pragma unroll
                    for (int j = 0; j < CPL; ++j) d[dzhi + j] = out[i][j];
                }
                if (xlo && oo[i] == 0) d[dxlo] = out[i][0];
                if (xhi && oo[i] == 1) d[dxhi + CPL - 1] = out[i][CPL - 1];
            }
            kofs += cplane;
        }
        release(g + (uint32_t)nk + 1);
        g += (uint32_t)nk + 2;
    }
}

template <int CPL, int NWARP, int RPW>
int launch_split_one(const CUtensorMap &omap, const CUtensorMap &rmap, const SplitArgs &a, int nctas, size_t smem,
                     cudaStream_t s) {
    auto kern = split_pass_kernel<CPL, NWARP, RPW>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return tmk::cuda_fail(e, "cudaFuncSetAttribute(gsrb split)");
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nctas);
    cfg.blockDim = dim3((NWARP + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, omap, rmap, a);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "gsrb split launch");
    return TM_OK;
}

int encode_colour_map(CUtensorMap *map, const ColourLayout &C, const double *base, int box_y) {
    return tmk::encode_plane_map_strided(map, base, C.wp, C.ny + 2, C.nz + 2, C.nslots, C.plane, C.slot,
                                         C.nx / 2 + 4, box_y);
}

int encode_colour_rhs_map(CUtensorMap *map, const ColourLayout &C, const double *base, int rows) {
    tm_layout X{};
    X.nslots = C.nslots;
    X.ncomp = 1;
    X.pitch = C.nx / 2;
    X.ny = C.ny;
    X.nz = C.nz;
    return tmk::encode_plane_map(map, X, base, C.nx / 2, rows);
}

}  // namespace

extern "C" {

int tm_gsrb_split(const tm_layout *phi_layout, const double *phi, int32_t nx, int32_t ny, int32_t nz,
                  const int32_t *d_parity, double *c0, double *c1, const tm_layout *rhs_layout, const double *rhs,
                  double *r0, double *r1, void *stream) {
    using namespace tmk;
    int rc = check_layout(phi_layout, "tm_gsrb_split");
    if (rc) return rc;
    if (rhs) {
        rc = check_layout(rhs_layout, "tm_gsrb_split(rhs)");
        if (rc) return rc;
    }
    if (!phi || !c0 || !c1 || !d_parity || nx % 4 || nx < 4 || phi_layout->nghost < 1 ||
        (rhs && (!r0 || !r1)))
        return fail(TM_ERR_INVALID, "tm_gsrb_split: bad arguments (nx must be a multiple of 4, nghost >= 1)");
    const ColourLayout C = colour_layout(phi_layout->nslots, nx, ny, nz);
    if ((int64_t)C.nslots * (nz + 2) * (ny + 2) >= ((int64_t)1 << 31))
        return fail(TM_ERR_INVALID, "tm_gsrb_split: too many rows");
    const tm_layout R = rhs ? *rhs_layout : *phi_layout;
    split_kernel<<<148 * 8, 256, 0, as_stream(stream)>>>(*phi_layout, phi, C, d_parity, c0, c1, R, rhs, r0, r1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TM_OK : cuda_fail(e, "tm_gsrb_split launch");
}

int tm_gsrb_merge(const tm_layout *phi_layout, double *phi, int32_t nx, int32_t ny, int32_t nz,
                  const int32_t *d_parity, const double *c0, const double *c1, void *stream) {
    using namespace tmk;
    int rc = check_layout(phi_layout, "tm_gsrb_merge");
    if (rc) return rc;
    if (!phi || !c0 || !c1 || !d_parity || nx % 4 || nx < 4)
        return fail(TM_ERR_INVALID, "tm_gsrb_merge: bad arguments");
    const ColourLayout C = colour_layout(phi_layout->nslots, nx, ny, nz);
    if ((int64_t)C.nslots * nz * ny >= ((int64_t)1 << 31)) return fail(TM_ERR_INVALID, "tm_gsrb_merge: too many rows");
    merge_kernel<<<148 * 8, 256, 0, as_stream(stream)>>>(*phi_layout, phi, C, d_parity, c0, c1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TM_OK : cuda_fail(e, "tm_gsrb_merge launch");
}

int tm_gsrb_split_pass(tm_march_plan *p, int32_t nslots, int32_t nx, int32_t ny, int32_t nz, int32_t color,
                       double h2, const double *other, double *cur, const double *rhs_c, const int32_t *d_nbr,
                       void *stream) {
    using namespace tmk;
    if (!p) return fail(TM_ERR_INVALID, "tm_gsrb_split_pass: null plan");
    if (!other || !cur || !rhs_c || !d_nbr || (color != 0 && color != 1) || nx % 4 || nx > 128)
        return fail(TM_ERR_INVALID, "tm_gsrb_split_pass: bad arguments");
    if (p->ncols == 0) return TM_OK;
    if (p->max_nx != nx || p->max_ny > 32) return fail(TM_ERR_INVALID, "tm_gsrb_split_pass: columns must span the box width, <= 32 rows");
    if (colour_layout(nslots, nx, ny, nz).plane * (int64_t)(nz + 2) >= ((int64_t)1 << 31))
        return fail(TM_ERR_INVALID, "tm_gsrb_split_pass: one slot of a colour array must hold < 2^31 doubles");
    SplitArgs a{};
    a.cols = p->d_cols;
    a.segs = p->d_segs;
    a.seg_begin = p->d_seg_begin;
    a.C = colour_layout(nslots, nx, ny, nz);
    a.out = cur;
    a.nbr = d_nbr;
    a.color = color;
    a.h2 = h2;
    a.box_y = p->max_ny + 2;
    a.rhs_off = (((a.C.nx / 2 + 4) * a.box_y + 15) / 16) * 16;
    a.stage_elems = a.rhs_off + ((nx / 2 * p->max_ny + 15) / 16) * 16;
    const size_t smem = (size_t)kSStages * a.stage_elems * sizeof(double) + 2 * kSStages * sizeof(uint64_t);
    if (smem > 220 * 1024)
        return fail(TM_ERR_INVALID, "tm_gsrb_split_pass: column plane too large for the shared-memory ring (use "
                                    "fewer rows per column)");
    CUtensorMap omap, rmap;
    int rc = encode_colour_map(&omap, a.C, other, a.box_y);
    if (rc) return rc;
    rc = encode_colour_rhs_map(&rmap, a.C, rhs_c, p->max_ny);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    const int nh = nx / 2;
    if (nh <= 32) {
        if (p->max_ny <= 16) return launch_split_one<1, 8, 2>(omap, rmap, a, p->nctas, smem, s);
        return launch_split_one<1, 16, 2>(omap, rmap, a, p->nctas, smem, s);
    }
    if (p->max_ny <= 16) return launch_split_one<2, 8, 2>(omap, rmap, a, p->nctas, smem, s);
    return launch_split_one<2, 16, 2>(omap, rmap, a, p->nctas, smem, s);
}

}  // extern "C"
