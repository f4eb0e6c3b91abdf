/*
 * tilemesh_b200.h -- C ABI of libtilemesh_b200.so, the sm_100a kernels
 * behind the tilemesh stencil-sweep + FillBoundary hot path.
 *
 * The reference (/root/reference/pkg/src/tilemesh, Python + numba) has no
 * C ABI; its replaceable seam is the set of numba loop nests in compiled.py
 * plus the numpy tag copies of level.py.  Each entry point below replaces
 * one of them (file:line in the reference):
 *
 *   tm_copy_run            level.py:290-294   _run_tags (FillBoundary copies);
 *                          also halo pack/unpack for remote boxes and the
 *                          scatter/gather of domain arrays
 *   tm_heat_sweep          compiled.py:84-99  heat_tiles (flux_x/y/z :32-63
 *                          + divergence :66-81), driven as kernels.py:174-215
 *   tm_gsrb_color          (no reference kernel)
 *   tm_residual_maxnorm    (no reference kernel)
 *   tm_reduce_sum          level.py:183-190 + compiled.py:20-29 serial_sum
 *   tm_reduce_minmax       level.py:175-181 reduce_max / reduce_min
 *
 * Conventions:
 *   - every function returns 0 (TM_OK) or a TM_ERR_* code; the message is
 *     available from tm_last_error() (thread-local); no C++ exceptions
 *     cross the ABI;
 *   - device memory is owned by the caller (PyTorch allocations); the
 *     library only borrows pointers.  Plans are library-owned handles
 *     holding device copies of their tables;
 *   - `stream` is a cudaStream_t passed as void*; calls are asynchronous on
 *     that stream, the caller synchronises;
 *   - no checks inside kernels (the reference's "unchecked fast path",
 *     SPEC.md:134); arguments are validated on the host before launch.
 *
 * Device storage of a MultiFab ("layout"): one fp64 allocation holding
 * nslots FAB slots; slot s, component c, plane z, row y, column x lives at
 *     base[((s*ncomp + c)*nz + z)*ny*pitch + y*pitch + x]
 * The grown box of a unit sits at slot origin with its first VALID cell at
 * column xoff (a multiple of 16 doubles = 128 B) and row/plane nghost, so
 * every valid i-row starts 128-B aligned; pitch is a multiple of 16.
 */
#ifndef TILEMESH_B200_H
#define TILEMESH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TM_OK 0
#define TM_ERR_INVALID 1 /* bad argument (reference raises ValueError) */
#define TM_ERR_CUDA 2    /* CUDA runtime / driver failure */
#define TM_ERR_NOMEM 3

#define TM_ABI_VERSION 4

typedef struct tm_layout {
    int64_t nslots; /* FAB slots in the allocation */
    int32_t ncomp;
    int32_t nghost;
    int32_t pitch; /* doubles per row, multiple of 16 */
    int32_t ny;    /* rows per plane  (>= max grown y extent) */
    int32_t nz;    /* planes per comp (>= max grown z extent) */
    int32_t xoff;  /* column of the first valid cell, multiple of 16 */
} tm_layout;

/* One rectangular copy of ex*ey*ez cells x ncomp components.  Offsets are
 * element offsets of the first cell (component 0) from the side's base. */
typedef struct tm_copy_tag {
    int64_t dst_off;
    int64_t src_off;
    int32_t ex, ey, ez;
    int32_t reserved;
} tm_copy_tag;

/* Addressing of one side of a copy: element strides of y, z and component.
 * sy == 0 means "packed": the tag's cells are contiguous in x,y,z,c order
 * (strides ex, ex*ey, ex*ey*ez) -- the halo send/receive buffer format. */
typedef struct tm_side {
    int64_t sy, sz, sc;
} tm_side;

/* One CTA work unit of a sweep: a tile of one FAB slot.  x0,y0,z0 are slot
 * coordinates of the tile's first cell; parity = (i+j+k)&1 of that cell in
 * global index space (red/black colouring). */
typedef struct tm_block {
    int32_t slot;
    int32_t x0, y0, z0;
    int32_t nx, ny, nz;
    int32_t parity;
} tm_block;

typedef struct tm_copy_plan tm_copy_plan;
typedef struct tm_sweep_plan tm_sweep_plan;

const char *tm_last_error(void);
int tm_abi_version(void);
/* sm_100a device present and usable (0) or TM_ERR_CUDA */
int tm_device_check(int device);

/* ---- FillBoundary / halo pack / unpack / scatter / gather ---------------- */
int tm_copy_plan_create(const tm_copy_tag *tags, int64_t ntags, int32_t ncomp, tm_copy_plan **out);
int tm_copy_plan_destroy(tm_copy_plan *plan);
int64_t tm_copy_plan_elements(const tm_copy_plan *plan); /* cells x ncomp */
int tm_copy_run(const tm_copy_plan *plan, double *dst, const tm_side *dst_side, const double *src,
                const tm_side *src_side, void *stream);
/* x-face ghosts (one ghost layer, valid y/z range) of every slot from a
 * packed x-halo buffer xh[(slot*ncomp+c)][z][side][y] as tm_heat_march writes
 * it for a field (side 0 -> x = lo-1, side 1 -> x = hi+1; uniform valid x
 * extent nx; nghost == 1).  Each ghost is written as a whole 64-B chunk of its
 * row (the ghost plus row padding nothing reads).  The x-face part of
 * fill_boundary (level.py:297-323) for a field whose packed halos are known. */
int tm_xh_to_ghosts(const tm_layout *layout, double *base, const double *xh, int32_t nx, void *stream);

/* ---- stencil sweeps -------------------------------------------------------- */
int tm_sweep_plan_create(const tm_block *blocks, int64_t nblocks, tm_sweep_plan **out);
int tm_sweep_plan_destroy(tm_sweep_plan *plan);

/* unew = uold + dtD*div(grad uold) on every block cell, components
 * [comp0, comp0+ncomp_sweep).  Requires uold ghosts (1 layer) filled. */
int tm_heat_sweep(tm_sweep_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                  int32_t comp0, int32_t ncomp_sweep, double dxi0, double dxi1, double dxi2,
                  double dtD, void *stream);

/* In-place red (color 0) or black (color 1) Gauss-Seidel update of phi
 * (component 0) for -lap(phi) = rhs; h2 = dx*dx. */
int tm_gsrb_color(tm_sweep_plan *plan, const tm_layout *phi_layout, double *phi,
                  const tm_layout *rhs_layout, const double *rhs, int32_t color, double h2,
                  void *stream);

/* d_out[0] = max |rhs + (sum6(phi) - 6 phi)/h2| over block cells (device
 * double, overwritten). */
int tm_residual_maxnorm(tm_sweep_plan *plan, const tm_layout *phi_layout, const double *phi,
                        const tm_layout *rhs_layout, const double *rhs, double h2, double *d_out,
                        void *stream);

/* ---- persistent column-march heat sweep (Kernel A2) -------------------------
 * Replaces the same reference call as tm_heat_sweep (compiled.py:84-99 via
 * kernels.py:174-215) with a different CTA decomposition: `columns` are box
 * tiles spanning the full z extent (tm_block with nz = box nz); `nctas`
 * persistent CTAs each march an equal share of all column planes.
 * Columns must start on an even x and have even width <= 128, height <= 64. */
typedef struct tm_march_plan tm_march_plan;
int tm_march_plan_create(const tm_block *columns, int64_t ncolumns, int32_t nctas, tm_march_plan **out);
int tm_march_plan_destroy(tm_march_plan *plan);
/* Where a step's halos come from, and which halos of the new field it writes
 * (halo_mode of tm_heat_march):
 *   TM_HALO_GHOSTS        x/y/z halos from the ghost cells of uold (FillBoundary
 *                         must have run); writes only valid cells of unew.
 *                         xh_old, xh_new, d_nbr must be NULL, reverse 0.
 *   TM_HALO_GHOSTS_XH     as GHOSTS (halos read from uold's ghost cells), and the
 *                         epilogue also writes the packed x halos of unew's
 *                         boxes into xh_new (d_nbr as below): unew's storage
 *                         is written on valid cells only -- the reference's
 *                         heat_step contract -- and the next step may take its
 *                         x halos from xh_new.
 *   TM_HALO_PACKED        x halos from the packed buffer xh_old
 *                         xh[(slot*ncomp+c)][z][side][y] (valid y,z extents;
 *                         side 0 = i = lo-1, side 1 = i = hi+1), y/z from the
 *                         ghosts of uold; writes only valid cells of unew.
 *   TM_HALO_FUSED_SCATTER as PACKED, and the epilogue also writes every box's
 *                         boundary values into its face neighbours' halos of
 *                         the new field: y/z ghost rows/planes of unew and the
 *                         packed x halo xh_new (d_nbr: 6 neighbour slots per
 *                         slot, order -x,+x,-y,+y,-z,+z; < 0 = none / remote).
 *   TM_HALO_FUSED_NBR     y/z halos read straight from the face neighbours'
 *                         valid cells in uold (own ghosts where d_nbr < 0),
 *                         x halos from xh_old; the epilogue writes ONLY xh_new.
 *                         The y/z face ghosts of unew are NOT written.  Needs
 *                         columns of one height and width % 16 == 0.
 *   TM_HALO_FUSED_NBR_GHOSTS  as FUSED_NBR (forward, nghost 1), and the y/z
 *                         halo rows and planes it loads -- exactly the y/z face
 *                         ghosts of uold a FillBoundary writes -- are also
 *                         stored into uold's ghosts (faces with a local
 *                         neighbour): the y/z face part of a preceding
 *                         fill_boundary, deferred into the sweep.  The only
 *                         mode that writes through `uold`.
 * The fused modes are the FillBoundary of the next step fused into this one
 * (face halos only: the 7-point stencil never reads edge/corner ghosts).  A
 * SCATTER step must not follow an NBR step on the same packed halos (the y/z
 * ghosts it reads were not written): the plan remembers the last fused mode
 * and refuses that hand-over until tm_march_plan_reset_halos (call it after
 * re-priming the halos with a FillBoundary).
 * reverse != 0 (fused modes): every CTA walks its columns in reverse order and
 * marches z downward -- same results; a step that follows a forward step then
 * starts on the planes that step wrote last (L2-resident).
 * Launched with programmatic stream serialization (PDL): the kernel's prologue
 * may overlap the previous kernel on the stream; it waits (griddepcontrol.wait)
 * for that kernel to complete before touching uold/unew, so stream order is
 * preserved. */
enum {
    TM_HALO_GHOSTS = 0,
    TM_HALO_PACKED = 1,
    TM_HALO_FUSED_SCATTER = 2,
    TM_HALO_FUSED_NBR = 3,
    TM_HALO_GHOSTS_XH = 4,
    TM_HALO_FUSED_NBR_GHOSTS = 5
};
int tm_heat_march(tm_march_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                  int32_t ncomp_sweep, double dxi0, double dxi1, double dxi2, double dtD, int32_t halo_mode,
                  const double *xh_old, double *xh_new, const int32_t *d_nbr, int32_t reverse, void *stream);
/* The reference-shaped loop's step on the fast path (fill_boundary, level.py:297-323, then
 * heat_step, kernels.py:174-215, when the fill left uold's y/z face ghosts pending): the
 * TM_HALO_FUSED_NBR_GHOSTS sweep plus the fill's remaining cells -- uold's edge/corner ghosts,
 * d_fill_cells = device int64 pairs (dst, src) of element offsets from uold, copied from
 * uold's valid cells, which this launch does not write -- run by one extra warp per CTA while
 * the others march: one launch for the whole loop step. */
int tm_heat_march_fill(tm_march_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                       int32_t ncomp_sweep, double dxi0, double dxi1, double dxi2, double dtD, const double *xh_old,
                       double *xh_new, const int32_t *d_nbr, const int64_t *d_fill_cells, int64_t nfill_cells,
                       void *stream);
int tm_march_plan_reset_halos(tm_march_plan *plan);

/* Fused red (0) / black (1) Gauss-Seidel pass of the column march, in place on
 * phi (ncomp 1), x halos from the packed buffer xh, and the updated colour's
 * boundary values scattered into the face neighbours' halos (phi ghost
 * rows/planes and xh): the FillBoundary that follows each colour in
 * BASELINE config 4 is fused.  Same per-cell form as tm_gsrb_color. */
int tm_gsrb_march(tm_march_plan *plan, const tm_layout *phi_layout, double *phi, const tm_layout *rhs_layout,
                  const double *rhs, int32_t color, double h2, double *xh, const int32_t *d_nbr, void *stream);

/* ---- GSRB on colour-split storage (during a solve) ---------------------------
 * Each colour of phi in its own array [slot][z+1][y+1][i+4] (rows nx/2 + 8
 * doubles, so valid entries start on 32-B sectors; entry i of row (y, z) =
 * cell x = 2i + ((c + parity + y + z) & 1),
 * i in [-1, nx/2]), rhs split into [slot][z][y][nx/2] per colour.  A colour
 * pass reads only the other colour and writes only its own: 24 bytes per
 * UPDATED cell.  Same per-cell form as tm_gsrb_color (bit-identical); the
 * pass also fills the face neighbours' ghost entries of its colour.
 * d_parity[slot] = (x_lo + y_lo + z_lo) & 1 of each box; uniform boxes,
 * nx % 4 == 0. */
int tm_gsrb_split(const tm_layout *phi_layout, const double *phi, int32_t nx, int32_t ny, int32_t nz,
                  const int32_t *d_parity, double *c0, double *c1, const tm_layout *rhs_layout, const double *rhs,
                  double *r0, double *r1, void *stream);
int tm_gsrb_merge(const tm_layout *phi_layout, double *phi, int32_t nx, int32_t ny, int32_t nz,
                  const int32_t *d_parity, const double *c0, const double *c1, void *stream);
int tm_gsrb_split_pass(tm_march_plan *plan, int32_t nslots, int32_t nx, int32_t ny, int32_t nz, int32_t color,
                       double h2, const double *other, double *cur, const double *rhs_c, const int32_t *d_nbr,
                       void *stream);

/* ---- 9-point 8th-order Laplacian step ("wide4", Kernel W) -------------------
 * Replaces compiled.wide4_tiles / wide4_range (compiled.py:102-141) as driven
 * by kernels.wide4_step (kernels.py:218-247) and the reference's loop variant
 * (kernels.py:309-342), over every column of a march plan (columns of the
 * full box width <= 128, <= 16 rows (<= 8 when wider than 64), full z; or, on
 * Kernel W2, widths <= 64 with row counts that are multiples of 4, <= 32).
 * coeffs5 = host array {c0, c1, c2, c3, c4} (StencilCoeffs8); dxi2_d = 1/dx_d^2;
 * dtD = D*dt.  Needs nghost >= 4 with filled ghosts (FillBoundary).  Per cell,
 * in the reference's operation order, FMA-free: bit-identical. */
int tm_wide4_march(tm_march_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                   int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                   double dtD, void *stream);
/* Same step with FillBoundary fused into its epilogue (no reference
 * counterpart: replaces the fill_boundary + wide4_step pair of the
 * reference's step loop, level.py:297-323 + kernels.py:218-247, for uniform
 * fully-covered box layouts): every cell within 4 of a box face is also
 * written into the face neighbour's ghost layers of unew, so the next step's
 * x/y/z face ghosts are filled on return (edge/corner ghosts are not: the
 * stencil never reads them).  d_nbr = device int32[nslots][6] face neighbours
 * (-x,+x,-y,+y,-z,+z; local slot, < 0: none); box_extents = host int32[3],
 * the uniform box size (each >= 8). */
int tm_wide4_march_fused(tm_march_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                         int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                         double dtD, const int32_t *d_nbr, const int32_t *box_extents, void *stream);
/* The reference step loop's pair (fill_boundary, level.py:297-323 + wide4_step,
 * kernels.py:218-247) as ONE launch that writes nothing but unew's valid cells:
 * every x/y/z halo (4 deep) is read straight from the face neighbour's valid
 * cells of uold -- the values a FillBoundary would have copied -- so neither
 * field's ghosts are read or written (faces with no neighbour, d_nbr < 0, read
 * uold's own ghosts).  Needs uniform boxes whose width is a multiple of 4 and
 * <= 64, cut into full-width columns of one height (a multiple of 4, <= 32,
 * dividing the box height); each box extent >= 4.  Kernel W2 (tm_wide4.cu).
 * tm_wide4_march runs W2 too (halos from ghosts) when its plan allows. */
int tm_wide4_march_nbr(tm_march_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                       int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                       double dtD, const int32_t *d_nbr, const int32_t *box_extents, void *stream);
/* The reference loop's wide4 step on the fast path (fill_boundary with 4 ghost layers,
 * level.py:297-323, then wide4_step, kernels.py:218-247, when the fill was deferred): the
 * tm_wide4_march_nbr step that also writes every 4-deep face ghost of uold as it loads it from
 * the neighbours, plus the fill's edge/corner cells (d_fill_cells: device int64 (dst, src)
 * offset pairs from uold, one per run of 4 doubles along x, each 32-B aligned) copied by the
 * producer warpgroup's idle warps.  Needs nghost == 4. */
int tm_wide4_march_fill(tm_march_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                        int32_t ncomp_sweep, const double *coeffs5, double dxi2_0, double dxi2_1, double dxi2_2,
                        double dtD, const int32_t *d_nbr, const int32_t *box_extents, const int64_t *d_fill_cells,
                        int64_t nfill_cells, void *stream);

/* ---- per-tile heat operations (the reference's building blocks) -------------
 * tm_face_flux replaces heat_flux (kernels.py:86-120 -> compiled.flux_x/y/z,
 * compiled.py:32-63): out[f] = (u[f] - u[f - e_dir]) * dxi for the nx*ny*nz faces
 * of a face box; `u` points at the high cell of face (0,0,0).
 * tm_divergence_update replaces heat_divergence_update (kernels.py:122-144 ->
 * compiled.divergence, compiled.py:66-81): on the nx*ny*nz cells of a tile,
 * unew = uold + dtD*(((fx[+1]-fx)*dxi0 + (fy[+1]-fy)*dxi1) + (fz[+1]-fz)*dxi2)
 * with fx/fy/fz indexed from the tile's first cell.  All arrays are strided
 * views with x contiguous (strides of y and z in elements).  FMA-free, the
 * reference's operation order: bit-identical. */
int tm_face_flux(const double *u, int64_t u_sy, int64_t u_sz, int32_t direction, int32_t nx, int32_t ny,
                 int32_t nz, double dxi, double *out, int64_t out_sy, int64_t out_sz, void *stream);
int tm_divergence_update(double *unew, const double *uold, int64_t u_sy, int64_t u_sz, const double *fx,
                         int64_t fx_sy, int64_t fx_sz, const double *fy, int64_t fy_sy, int64_t fy_sz,
                         const double *fz, int64_t fz_sy, int64_t fz_sz, int32_t nx, int32_t ny, int32_t nz,
                         double dxi0, double dxi1, double dxi2, double dtD, void *stream);

/* ---- reductions (one block per unit, blocks in grid order) --------------- */
/* d_partial[b] = serial x-fastest sum of block b (from 0.0); d_total[0] =
 * serial sum of the partials in block order: bit-identical to the
 * reference reduce_sum. d_partial needs nblocks doubles. */
int tm_reduce_sum(tm_sweep_plan *plan, const tm_layout *layout, const double *base, int32_t comp,
                  double *d_partial, double *d_total, void *stream);
/* d_out[0] = max, d_out[1] = min over block cells of component comp. */
int tm_reduce_minmax(tm_sweep_plan *plan, const tm_layout *layout, const double *base, int32_t comp,
                     double *d_out, void *stream);

/* ---- inter-GPU halo exchange (NCCL) ----------------------------------------
 * Replaces the remote half of fill_boundary (level.py:297-323) when boxes live
 * on several GPUs (one process per GPU): pack the outgoing
 * ghost data with tm_copy_run (packed side), move every message of the fill
 * with ONE grouped ncclSend/ncclRecv to the neighbour ranks only, unpack with
 * tm_copy_run.  BoxLib's aggregated remote-ghost buffers: PAPER.md:303-314.
 * NCCL is dlopen'ed (an already loaded libnccl.so.2 is reused; TM_NCCL_LIB
 * overrides the path).  tm_comm_create binds to the current CUDA device; the
 * caller shares the 128-byte unique id of rank 0 (e.g. through the
 * torch.distributed store) at setup only.  tm_halo_exchange is asynchronous
 * on `stream` and may be captured into a CUDA graph. */
typedef struct tm_comm tm_comm;
typedef struct tm_exchange tm_exchange;
int tm_comm_nccl_version(int32_t *version);
int tm_comm_unique_id(uint8_t *out128);
int tm_comm_create(const uint8_t *id128, int32_t nranks, int32_t rank, tm_comm **out);
int tm_comm_destroy(tm_comm *comm);
/* npeers distinct ascending peer ranks; message i: send_count[i] doubles at
 * sendbuf + send_off[i] to peers[i], recv_count[i] doubles from peers[i] into
 * recvbuf + recv_off[i] (counts may be 0 on either side). */
int tm_exchange_create(tm_comm *comm, int32_t npeers, const int32_t *peers, const int64_t *send_off,
                       const int64_t *send_count, const int64_t *recv_off, const int64_t *recv_count,
                       tm_exchange **out);
int tm_exchange_destroy(tm_exchange *x);
int tm_halo_exchange(tm_exchange *x, const double *sendbuf, double *recvbuf, void *stream);

/* ---- peer (NVLink / NVSwitch) halos: the exchange fused into the sweep -----
 * Replaces the remote half of fill_boundary (level.py:297-323) together with
 * the heat_step that follows it (kernels.py:174-215) when the GPUs of the job
 * can map each other's memory: the march kernel (TM_HALO_FUSED_NBR) TMA-loads
 * the y/z halo planes and rows of a box whose face neighbour lives on another
 * rank straight from that rank's valid cells over NVLink, plane by plane while
 * it computes.  No pack, no message, no unpack; a step is one march launch
 * plus one tm_peer_barrier.  BoxLib's remote ghost traffic: PAPER.md:549-556.
 *
 * Neighbour table entries (d_nbr, 6 per slot) for faces on another rank:
 * TM_NBR_PEER(p, s) = -3 - (p * 2^24 + s): slot s of peer p of the current
 * peer set (p < TM_MAX_PEERS, s < 2^24).  Only y and z faces may be peers (x
 * neighbours stay on the rank: the packed x halos are written locally).
 *
 * tm_ipc_export: a CUDA IPC handle (64 bytes) of the allocation holding ptr
 * and ptr's byte offset inside it.  tm_ipc_open (in another process) maps it
 * and returns the peer's ptr; tm_ipc_close unmaps (pass the pointer
 * tm_ipc_open returned).
 *
 * tm_march_plan_set_peers: peer set `set` (< TM_PEER_SETS) = npeers fields,
 * peer p's storage at peer_base[p] with the caller's layout except nslots =
 * peer_nslots[p] (every rank of a job shares pitch / ny / nz / xoff / ncomp /
 * nghost).  Encodes the peers' TMA maps once into device memory; call at
 * setup, not inside a graph capture.  A double-buffered pair uses set 0 for
 * the peers' first field and set 1 for their second.
 *
 * tm_heat_march_peer: tm_heat_march in TM_HALO_FUSED_NBR with peer faces read
 * through `set`.  The peers' uold must be complete and the peers must have
 * finished reading the field unew overwrites (their previous step): order the
 * ranks with one tm_peer_barrier between consecutive steps.
 *
 * tm_peer_barrier: device-side barrier of this rank with `npeers` peers on
 * `stream`, graph-capturable.  inbox = this rank's TM_MAX_RANKS uint64
 * counters (device memory, zeroed once; peers hold it through IPC),
 * peer_inbox[i] = rank peer_ranks[i]'s inbox as mapped here (device array of
 * pointers), epoch = this rank's uint64 epoch counter (device).  One thread
 * per peer adds 1 to peer_inbox[i][my_rank] (release, system scope), then
 * waits until inbox[peer_ranks[i]] reaches the new epoch (acquire, system
 * scope).  A wait that exceeds timeout_ns sets *status (device int32) to 1
 * and returns instead of hanging.  Only for ranks on DIFFERENT GPUs: ranks
 * sharing a GPU must be ordered by the host (B200_PROFILING.md: kernels that
 * wait on one another must not share a device). */
#define TM_MAX_PEERS 8
#define TM_PEER_SETS 4
#define TM_MAX_RANKS 64
#define TM_NBR_PEER(p, s) (-3 - (int32_t)(((int32_t)(p) << 24) + (int32_t)(s)))
int tm_ipc_export(const void *ptr, uint8_t *handle64, int64_t *offset);
int tm_ipc_open(const uint8_t *handle64, int64_t offset, void **ptr);
int tm_ipc_close(void *ptr, int64_t offset);
int tm_march_plan_set_peers(tm_march_plan *plan, int32_t set, const tm_layout *layout, int32_t npeers,
                            const double *const *peer_base, const int64_t *peer_nslots);
int tm_heat_march_peer(tm_march_plan *plan, const tm_layout *layout, const double *uold, double *unew,
                       int32_t ncomp_sweep, double dxi0, double dxi1, double dxi2, double dtD, const double *xh_old,
                       double *xh_new, const int32_t *d_nbr, int32_t set, int32_t reverse, void *stream);
int tm_peer_barrier(uint64_t *inbox, uint64_t *const *peer_inbox, const int32_t *peer_ranks, int32_t npeers,
                    int32_t my_rank, uint64_t *epoch, int32_t *status, int64_t timeout_ns, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TILEMESH_B200_H */
