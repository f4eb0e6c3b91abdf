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

constexpr int kSStages = 4;

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
    C.wp = nx / 2 + 8;
    C.row = C.wp;
    C.plane = C.row * (ny + 2);
    C.slot = C.plane * (nz + 2);
    C.rrow = nx / 2;
    C.rplane = C.rrow * ny;
    C.rslot = C.rplane * nz;
    return C;
}

// phi (valid + one ghost layer) -> both colour arrays; rhs -> both colour rhs arrays
__global__ void split_kernel(tm_layout L, const double *__restrict__ phi, ColourLayout C, const int32_t *parity,
                             double *__restrict__ c0, double *__restrict__ c1, tm_layout R,
                             const double *__restrict__ rhs, double *__restrict__ r0, double *__restrict__ r1) {
    const int nh = C.nx / 2;
    const int64_t rows = (int64_t)C.nslots * (C.nz + 2) * (C.ny + 2);
    const tmk::Strides s = tmk::strides_of(L);
    const tmk::Strides rs = tmk::strides_of(R);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.y + threadIdx.y; t < rows; t += (int64_t)gridDim.x * blockDim.y) {
        const int yy = (int)(t % (C.ny + 2)), zz = (int)((t / (C.ny + 2)) % (C.nz + 2));
        const int slot = (int)(t / ((int64_t)(C.ny + 2) * (C.nz + 2)));
        const int y = yy - 1, z = zz - 1;
        const double *prow = phi + slot * s.slot + (int64_t)(z + L.nghost) * s.plane + (int64_t)(y + L.nghost) * s.row +
                             L.xoff;
        const bool valid_row = y >= 0 && y < C.ny && z >= 0 && z < C.nz;
        for (int i = (int)threadIdx.x - 1; i <= nh; i += blockDim.x) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int o = (c + parity[slot] + y + z) & 1;
                const int x = 2 * i + o;
                double *dst = (c ? c1 : c0) + slot * C.slot + (int64_t)zz * C.plane + (int64_t)yy * C.row + (i + kE0);
                if (x >= -1 && x <= C.nx) *dst = prow[x];
                if (rhs && valid_row && i >= 0 && i < nh) {
                    const double *rrow = rhs + slot * rs.slot + (int64_t)(z + R.nghost) * rs.plane +
                                         (int64_t)(y + R.nghost) * rs.row + R.xoff;
                    (c ? r1 : r0)[slot * C.rslot + (int64_t)z * C.rplane + (int64_t)y * C.rrow + i] = rrow[x];
                }
            }
        }
    }
}

// both colour arrays -> phi valid cells
__global__ void merge_kernel(tm_layout L, double *__restrict__ phi, ColourLayout C, const int32_t *parity,
                             const double *__restrict__ c0, const double *__restrict__ c1) {
    const int nh = C.nx / 2;
    const int64_t rows = (int64_t)C.nslots * C.nz * C.ny;
    const tmk::Strides s = tmk::strides_of(L);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.y + threadIdx.y; t < rows; t += (int64_t)gridDim.x * blockDim.y) {
        const int y = (int)(t % C.ny), z = (int)((t / C.ny) % C.nz);
        const int slot = (int)(t / ((int64_t)C.ny * C.nz));
        double *prow = phi + slot * s.slot + (int64_t)(z + L.nghost) * s.plane + (int64_t)(y + L.nghost) * s.row + L.xoff;
        for (int i = threadIdx.x; i < nh; i += blockDim.x) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int o = (c + parity[slot] + y + z) & 1;
                prow[2 * i + o] =
                    (c ? c1 : c0)[slot * C.slot + (int64_t)(z + 1) * C.plane + (int64_t)(y + 1) * C.row + (i + kE0)];
            }
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
    __syncthreads();

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
    uint32_t g = 0;
    for (int s = s_begin; s < s_end; ++s) {
        const Segment sg = a.segs[s];
        const tm_block c = a.cols[sg.col];
        const int nk = sg.k1 - sg.k0;
        const int yv0 = c.y0 - 1, zv0 = c.z0 - 1 + sg.k0;  // valid y of row 0, valid z of the first plane
        // neighbour slot deltas in registers (the scatter stores could alias a global table)
        int64_t dn[6];
        bool hn[6];
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            const int32_t t = a.nbr[6 * c.slot + f];
            hn[f] = t >= 0;
            dn[f] = (int64_t)(t - c.slot) * C.slot;
        }
        dn[0] += nh;                        // x = 0 -> -x neighbour's entry nh
        dn[1] -= nh;                        // x = nx-1 -> +x neighbour's entry -1
        dn[2] += (int64_t)C.ny * C.row;     // row 0 -> -y neighbour's row ny
        dn[3] -= (int64_t)C.ny * C.row;     // row ny-1 -> +y neighbour's row -1
        dn[4] += (int64_t)C.nz * C.plane;   // plane 0 -> -z neighbour's plane nz
        dn[5] -= (int64_t)C.nz * C.plane;   // plane nz-1 -> +z neighbour's plane -1
        const bool lane_on = lane * CPL < nh;
        const int ii = min(lane * CPL, nh - CPL);  // lane's first entry
        int rr[RPW];
        bool on[RPW];
        uint32_t so[RPW], ro[RPW];  // stage byte offsets: other colour at (row, entry ii), rhs
        double *orow[RPW];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int r = warp * RPW + i;
            rr[i] = r;
            on[i] = lane_on && r < c.ny;
            const int rc = min(r, R - 1);
            so[i] = (uint32_t)((rc + 1) * wp + ii + 2) * 8u;
            ro[i] = (uint32_t)(a.rhs_off + rc * nh + ii) * 8u;
            orow[i] = a.out + c.slot * C.slot + (int64_t)(yv0 + r + 1) * C.row + (ii + kE0);
        }
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
        for (int kk = 0; kk < nk; ++kk) {
            const uint32_t gc = g + 1 + (uint32_t)kk;
            wait_plane(gc + 1);
            const uint32_t sc = saddr(gc), sn = saddr(gc + 1);
            const int zv = zv0 + kk;
            double out[RPW][CPL];
#pragma unroll
            for (int i = 0; i < RPW; ++i) {
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    const int o = (a.color + c.parity + rr[i] + sg.k0 + kk) & 1;
                    const uint32_t p = sc + so[i] + 8u * j;
                    const double w = lds_f64(p - 8u + 8u * o), e = lds_f64(p + 8u * o);
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
                double *d = orow[i] + (int64_t)(zv + 1) * C.plane;
#pragma unroll
                for (int j = 0; j < CPL; ++j) d[j] = out[i][j];
                // fused FillBoundary of this colour: face neighbours' ghost entries
                const int yv = yv0 + rr[i];
                const int o = (a.color + c.parity + rr[i] + sg.k0 + kk) & 1;
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    const int e_i = ii + j;
                    if (o == 0 && e_i == 0 && hn[0]) d[j + dn[0]] = out[i][j];
                    if (o == 1 && e_i == nh - 1 && hn[1]) d[j + dn[1]] = out[i][j];
                }
                const bool sy = (yv == 0 && hn[2]) || (yv == C.ny - 1 && hn[3]);
                if (sy) {
                    const int64_t dy = yv == 0 ? dn[2] : dn[3];
#pragma unroll
                    for (int j = 0; j < CPL; ++j) d[j + dy] = out[i][j];
                }
                const bool sz = (zv == 0 && hn[4]) || (zv == C.nz - 1 && hn[5]);
                if (sz) {
                    const int64_t dz = zv == 0 ? dn[4] : dn[5];
#pragma unroll
                    for (int j = 0; j < CPL; ++j) d[j + dz] = out[i][j];
                }
            }
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
    kern<<<nctas, (NWARP + 1) * 32, smem, s>>>(omap, rmap, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tmk::cuda_fail(e, "gsrb split launch");
    return TM_OK;
}

int encode_colour_map(CUtensorMap *map, const ColourLayout &C, const double *base, int box_y) {
    tm_layout X{};
    X.nslots = C.nslots;
    X.ncomp = 1;
    X.pitch = C.wp;
    X.ny = C.ny + 2;
    X.nz = C.nz + 2;
    return tmk::encode_plane_map(map, X, base, C.nx / 2 + 4, box_y);
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
    const tm_layout R = rhs ? *rhs_layout : *phi_layout;
    split_kernel<<<592, dim3(32, 8), 0, as_stream(stream)>>>(*phi_layout, phi, C, d_parity, c0, c1, R, rhs, r0, r1);
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
    merge_kernel<<<592, dim3(32, 8), 0, as_stream(stream)>>>(*phi_layout, phi, C, d_parity, c0, c1);
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
