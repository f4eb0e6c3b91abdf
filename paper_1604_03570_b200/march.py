"""Persistent column-march sweep (Kernel A2) and the fused halo path.

Host side of ``csrc/tm_march.cu``:

* ``march_columns`` cuts every local box into full-width x columns of at
  most ``max_rows`` rows spanning the whole box in z (the CTA work unit of
  the march kernel; results do not depend on the cut -- same arithmetic per
  cell as the reference, bit for bit);
* ``heat_march`` runs one sweep with x halos read from the ghost columns
  (after a regular FillBoundary);
* ``FusedHalo`` keeps packed x-halo buffers and a face-neighbour table for a
  pair of MultiFabs so that a step is ONE launch: the sweep reads face halos
  written by the previous step's epilogue and scatters its own boundary
  values into the neighbours' halos of the new field (the fused FillBoundary
  of SURVEY.md §7.9).  Edge/corner ghosts are not needed by the 7-point
  stencil and are only refreshed by ``finalize`` (a regular FillBoundary).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .box import Box
from .boxarray import BoxIndex, Geometry
from .multifab import MultiFab, cell_offsets

SMEM_BUDGET = 220 * 1024
STAGES = 4        # heat ring depth (tm_march.cu kHeatStages)
GSRB_STAGES = 4   # GSRB ring depth (kGsrbStages)


def sm_count(device) -> int:
    import torch

    return torch.cuda.get_device_properties(device).multi_processor_count


def _even_chunks(n: int, cap: int) -> list:
    """Split n into ceil(n/cap) near-equal EVEN chunks (n even)."""
    parts = -(-n // cap)
    pairs = n // 2
    q, r = divmod(pairs, parts)
    out = []
    pos = 0
    for p in range(parts):
        sz = 2 * (q + (p < r))
        out.append((pos, sz))
        pos += sz
    return out


CELLS_PER_PLANE = 1024  # column rows x width per CTA plane; C2 optimum (16 x 64), tools/march_perf.py


def warps_for(nx: int, rows: int) -> int:
    """Consumer warps of the heat / GSRB march kernel instance (mirrors launch_march)."""
    if nx > 64:  # 4 cells per lane
        return 8 if rows <= 8 else 16
    if nx > 32:  # 2 cells per lane
        return 4 if rows <= 8 else (7 if rows <= 14 else (8 if rows <= 16 else 16))
    if nx > 16 and rows <= 32:  # heat: half-warp row groups, 2 cells per lane (4 rows per warp)
        return 4 if rows <= 16 else 8
    return 4 if rows <= 8 else (8 if rows <= 32 else 16)  # 1 cell per lane


def max_rows_for(nx: int, packed: bool) -> int:
    width = nx if packed else nx + 4
    per_stage = SMEM_BUDGET // STAGES // 8 - (2 * 64 if packed else 0)
    rows = min(per_stage // width - 2, max(2, CELLS_PER_PLANE // nx), 64 if nx <= 64 else 32)
    return max(2, rows - rows % 2)


def march_eligible(mf: MultiFab) -> bool:
    L = mf.layout
    if mf.nghost < 1 or not mf.local_units:
        return False
    widths = [mf.units[u].valid.extents[0] for u in mf.local_units]
    if any(nx % 2 or nx > 128 for nx in widths):
        return False
    # columns wider than 64 run 4 cells per lane: the widest must be a multiple of 4
    # (tm_heat_march / tm_gsrb_march); other layouts take the tile kernel
    if max(widths) > 64 and max(widths) % 4:
        return False
    return L.xoff % 2 == 0


def march_columns(mf: MultiFab, max_rows: int | None = None, packed: bool = False) -> np.ndarray:
    L = mf.layout
    rows = []
    for u in mf.local_units:
        v = mf.units[u].valid
        nx, ny, nz = v.extents
        cap = max_rows or max_rows_for(nx, packed)
        if ny % 2 == 0:
            chunks = _even_chunks(ny, cap)
        else:
            if packed:
                raise ValueError("packed x halos need boxes of even y extent")
            n = -(-ny // cap)
            base, rem = divmod(ny, n)
            chunks, pos = [], 0
            for p in range(n):
                sz = base + (p < rem)
                chunks.append((pos, sz))
                pos += sz
        s = mf.slot_of[u]
        for (y0, sz) in chunks:
            rows.append((s, L.xoff, L.nghost + y0, L.nghost, nx, sz, nz, (v.lo[0] + v.lo[1] + y0 + v.lo[2]) & 1))
    out = np.zeros(len(rows), dtype=_native.BLOCK_DTYPE)
    arr = np.array(rows, dtype=np.int64).reshape(-1, 8)
    for n, name in enumerate(_native.BLOCK_DTYPE.names):
        out[name] = arr[:, n]
    return out


def ctas_per_sm(mf: MultiFab, columns: np.ndarray, packed: bool, rhs_rows: bool = False) -> int:
    nx = int(columns["nx"].max())
    ny = int(columns["ny"].max())
    width = nx if packed else nx + 4
    stage = -(-(width * (ny + 2)) // 16) * 16 + (-(-2 * ny // 16) * 16 if packed else 0)
    if rhs_rows:  # GSRB stages also carry the column's rhs rows
        stage += -(-(nx * ny) // 16) * 16
    smem = (GSRB_STAGES if rhs_rows else STAGES) * stage * 8 + 128
    threads = 32 * (1 + warps_for(nx, ny))
    return max(1, min(228 * 1024 // (smem + 1024), 2048 // threads, 65536 // (threads * 100)))


def march_plan(mf: MultiFab, packed: bool = False, max_rows: int | None = None,
               nctas: int | None = None, rhs_rows: bool = False, tag: str = "march") -> "_native.MarchPlan":
    key = (tag, packed, max_rows, nctas, rhs_rows, mf.layout, tuple(mf.local_units))
    plan = mf._plans.get(key)
    if plan is None:
        cols = march_columns(mf, max_rows, packed)
        n = nctas or sm_count(mf.device) * ctas_per_sm(mf, cols, packed, rhs_rows)
        plan = _native.MarchPlan(cols, n)
        mf._plans[key] = plan
    return plan


def heat_march(mf_new: MultiFab, mf_old: MultiFab, params, max_rows: int | None = None,
               nctas: int | None = None, geom: Geometry | None = None) -> None:
    """One sweep (all components); FillBoundary must have run, as for the
    reference's heat_step.  Bit-identical to heat_step.

    With ``geom`` and a one-rank layout of uniform boxes whose faces all have a
    neighbour box, the sweep also writes ``mf_new``'s packed x halos
    (``MultiFab.xh_buffer``: no storage cell beyond the valid ones), and when
    ``mf_old``'s packed x halos and ghosts are both current (the previous
    heat_step wrote the halos, a FillBoundary ran since, nothing else wrote the
    field) it reads y/z halos from the face neighbours' valid cells and x halos
    from the packed buffer -- the fused bench kernel -- instead of the ghost
    columns: the same values, fewer DRAM sectors.  ``fill_boundary`` likewise
    writes the x-face ghosts of a field with current packed halos from them."""
    if mf_old.nghost < 1:
        raise ValueError("heat kernel requires nghost >= 1")
    if not mf_new.same_layout(mf_old):
        raise ValueError("mf_new and mf_old must share box layout, ncomp, nghost and distribution")
    if not march_eligible(mf_old):
        raise ValueError("column march needs boxes of even x extent <= 128 (a multiple of 4 beyond 64)")
    c = params.coefficients()
    L = _native.load()
    route = xh_route(mf_old, geom) if geom is not None and max_rows is None and nctas is None else None
    if route is None:
        plan = march_plan(mf_old, False, max_rows, nctas)
        _native.check(L.tm_heat_march(plan.handle, mf_old.layout.to_c(), mf_old.ptr, mf_new.wptr,
                                      mf_old.ncomp, c[0], c[1], c[2], c[3], _native.HALO_GHOSTS,
                                      None, None, None, 0, mf_old.stream()), "tm_heat_march")
        return
    nbr, nbr_plan = route
    xh_new = mf_new.xh_buffer()  # not the buffer pinned as mf_new's deferred x face ghosts
    new_ptr = mf_new.wptr
    pending = mf_old._pending_faces
    if nbr_plan is not None and mf_old.xh_current() and (pending is not None or mf_old.ghosts_current()):
        plan, xh_old = nbr_plan, mf_old._xh.data_ptr()
        # a fill_boundary deferred mf_old's y/z face ghosts: this sweep writes them as it loads them
        mode = _native.HALO_FUSED_NBR if pending is None else _native.HALO_FUSED_NBR_GHOSTS
        old_ptr = mf_old._data.data_ptr()  # not .ptr: that would settle the pending faces first
        _native.check(L.tm_march_plan_reset_halos(plan.handle), "tm_march_plan_reset_halos")
    else:
        plan, mode, xh_old, old_ptr = march_plan(mf_old, False), _native.HALO_GHOSTS_XH, None, mf_old.ptr
    edges = mf_old._pending_edges if mode == _native.HALO_FUSED_NBR_GHOSTS else None
    if edges is not None:  # the fill's edge/corner cells ride on this launch (one extra warp per CTA)
        cells = mf_old._pending_cells
        _native.check(L.tm_heat_march_fill(plan.handle, mf_old.layout.to_c(), old_ptr, new_ptr, mf_old.ncomp,
                                           c[0], c[1], c[2], c[3], xh_old, xh_new.data_ptr(), nbr.data_ptr(),
                                           cells.data_ptr(), cells.shape[0], mf_old.stream()), "tm_heat_march_fill")
    else:
        _native.check(L.tm_heat_march(plan.handle, mf_old.layout.to_c(), old_ptr, new_ptr, mf_old.ncomp,
                                      c[0], c[1], c[2], c[3], mode, xh_old, xh_new.data_ptr(), nbr.data_ptr(), 0,
                                      mf_old.stream()), "tm_heat_march")
    mf_old._pending_edges = None
    mf_old._pending_faces = None
    mf_new._xh_key = mf_new.valid_key()


def default_fused_rows(mf: MultiFab):
    """Column height of the fused kernels: boxes wider than 64 run 4 cells per
    lane in 32-row columns, one 17-warp CTA per SM (C3, 128-wide boxes: 1.71
    -> 1.60 ms/step against 8-row columns at 2 CTAs/SM; tools/march_perf.py
    --config C3); otherwise ``max_rows_for``'s choice (None)."""
    return 32 if max(mf.units[u].valid.extents[0] for u in mf.local_units) > 64 else None


def xh_route(mf: MultiFab, geom: Geometry):
    """(face-neighbour table on the device, march plan of the neighbour-halo
    mode or None) when heat_step may keep packed x halos for this layout (one
    rank, fusable), else None.  Cached per MultiFab and geometry."""
    key = ("xh_route", geom)
    if key not in mf._plans:
        route = None
        if mf.dm.nranks == 1 and fusable(mf, geom):
            import torch

            table = face_neighbors(mf, geom)
            nbr = torch.as_tensor(table.reshape(-1), dtype=torch.int32, device=mf.device)
            plan = march_plan(mf, True, default_fused_rows(mf))
            cols = plan.columns
            ok = len(set(cols["ny"].tolist())) == 1 and int(cols["nx"].max()) % 16 == 0
            route = (nbr, plan if ok else None)
        mf._plans[key] = route
    return mf._plans[key]


# --------------------------------------------------------------------------
# fused halo path
# --------------------------------------------------------------------------
# --------------------------------------------------------------------------
# fused halo path
# --------------------------------------------------------------------------
REMOTE = -2  # face_neighbors entry: the neighbour lives on another rank


def face_neighbors(mf: MultiFab, geom: Geometry, allow_remote: bool = False):
    """Per local slot, the slots of the 6 face neighbours (-x,+x,-y,+y,-z,+z),
    or None when the layout is not fusable: every face must be covered by
    exactly one box of identical extents (uniform chopped domains, periodic
    or interior faces) that is LOCAL -- or, with ``allow_remote``, on another
    rank (entry ``REMOTE``: the kernels skip it, the halo exchange fills it)."""
    valids = [u.valid for u in mf.units]
    index = BoxIndex(valids)
    dom = geom.domain
    n = dom.extents
    table = np.full((len(mf.local_units), 6), -1, dtype=np.int32)
    for s, u in enumerate(mf.local_units):
        v = valids[u]
        e = v.extents
        for d in range(3):
            for side in (0, 1):
                shift = [0, 0, 0]
                shift[d] = -e[d] if side == 0 else e[d]
                lo = [v.lo[k] + shift[k] for k in range(3)]
                img = list(lo)
                if not (dom.lo[d] <= lo[d] and lo[d] + e[d] - 1 <= dom.hi[d]):
                    if not geom.periodic[d]:
                        return None
                    img[d] = dom.lo[d] + (lo[d] - dom.lo[d]) % n[d]
                target = Box(img, [img[k] + e[k] - 1 for k in range(3)])
                hits = index.query(target)
                if len(hits) != 1 or valids[hits[0]] != target:
                    return None
                nb = hits[0]
                if nb not in mf.slot_of:
                    if not allow_remote:
                        return None
                    table[s, 2 * d + side] = REMOTE
                    continue
                table[s, 2 * d + side] = mf.slot_of[nb]
    return table


def fusable(mf: MultiFab, geom: Geometry, allow_remote: bool = False) -> bool:
    if not march_eligible(mf):
        return False
    ext = {mf.units[u].valid.extents for u in mf.local_units}
    if len(ext) != 1:
        return False
    (nx, ny, nz), = ext
    L = mf.layout
    if ny % 2 or (L.ny - 2 * L.nghost) != ny or (L.nz - 2 * L.nghost) != nz:
        return False
    return face_neighbors(mf, geom, allow_remote) is not None


def xh_init_plan(mf: MultiFab, table, nyv: int, nzv: int):
    """Copy tags: each slot's two packed x halos <- the x-neighbours'
    boundary columns (valid y, z range, all components).  Returns
    (CopyPlan, packed-halo side strides)."""
    n = len(mf.local_units)
    slot_unit = np.array(mf.local_units, dtype=np.int64)
    vlo = np.array([mf.units[u].valid.lo for u in mf.local_units], dtype=np.int64).reshape(-1, 3)
    vhi = np.array([mf.units[u].valid.hi for u in mf.local_units], dtype=np.int64).reshape(-1, 3)
    ext = vhi - vlo + 1
    tags = np.zeros(2 * n, dtype=_native.COPY_TAG_DTYPE)
    for side in (0, 1):
        nb_slot = table[:, side].astype(np.int64)
        cells = vlo[nb_slot].copy()
        # left halo <- left neighbour's last column; right halo <- right neighbour's first
        cells[:, 0] = vhi[nb_slot, 0] if side == 0 else vlo[nb_slot, 0]
        src = cell_offsets(mf, slot_unit[nb_slot], cells)
        dst = ((np.arange(n, dtype=np.int64) * mf.ncomp) * nzv * 2 + side) * nyv
        t = tags[side::2]
        t["dst_off"], t["src_off"] = dst, src
        t["ex"], t["ey"], t["ez"] = 1, ext[:, 1], ext[:, 2]
    return _native.CopyPlan(tags, mf.ncomp), (1, 2 * nyv, 2 * nyv * nzv)


def xh_own_ghost_plan(mf: MultiFab, sides, nyv: int, nzv: int):
    """Copy tags: the packed x halo of (slot, side) <- the slot's own ghost
    column (x = -1 for side 0, x = nx for side 1), valid y and z, all
    components -- valid after a FillBoundary / halo exchange."""
    L = mf.layout
    tags = np.zeros(len(sides), dtype=_native.COPY_TAG_DTYPE)
    for t, (s, side) in enumerate(sides):
        nx = mf.units[mf.local_units[s]].valid.extents[0]
        src = s * L.slot + L.nghost * L.plane + L.nghost * L.row + (L.xoff - 1 if side == 0 else L.xoff + nx)
        dst = ((s * mf.ncomp) * nzv * 2 + side) * nyv
        tags[t] = (dst, src, 1, nyv, nzv, 0)
    return _native.CopyPlan(tags, mf.ncomp), (1, 2 * nyv, 2 * nyv * nzv)


def split_columns_by_sends(mf: MultiFab, cols: np.ndarray, send_src: dict):
    """Split march columns (full z extent) into (boundary, interior) column
    pieces along z: a piece is boundary when its planes hold cells that some
    send tag reads (``send_src``: unit -> source boxes, global indices).  A
    piece is a column with its own z range (tm_block z0 / nz), so both sets
    are ordinary march plans; every plane lands in exactly one of them."""
    L = mf.layout
    bnd, inner = [], []
    for c in cols:
        s, y0, z0, ny, nz = int(c["slot"]), int(c["y0"]), int(c["z0"]), int(c["ny"]), int(c["nz"])
        u = mf.local_units[s]
        v = mf.units[u].valid
        ylo = v.lo[1] + y0 - L.nghost
        zlo = v.lo[2] + z0 - L.nghost
        hit = np.zeros(nz, dtype=bool)
        for b in send_src.get(u, ()):
            if b.hi[1] < ylo or b.lo[1] > ylo + ny - 1:
                continue  # the column's rows miss this source box (columns span the full x extent)
            k0, k1 = max(b.lo[2] - zlo, 0), min(b.hi[2] - zlo, nz - 1)
            if k0 <= k1:
                hit[k0:k1 + 1] = True
        k = 0
        while k < nz:
            e = k
            while e < nz and hit[e] == hit[k]:
                e += 1
            piece = c.copy()
            piece["z0"], piece["nz"] = z0 + k, e - k
            (bnd if hit[k] else inner).append(piece)
            k = e
    mk = lambda rows: np.array(rows, dtype=_native.BLOCK_DTYPE) if rows else np.zeros(0, dtype=_native.BLOCK_DTYPE)  # noqa: E731
    return mk(bnd), mk(inner)


class FusedHalo:
    """Packed x halos + neighbour table shared by an old/new MultiFab pair."""

    def __init__(self, a: MultiFab, b: MultiFab, geom: Geometry, max_rows: int | None = None,
                 nctas: int | None = None, fill_plan=None):
        import torch

        from .multifab import comm_info

        multi = comm_info()[1] > 1
        if not (fusable(a, geom, multi) and a.same_layout(b)):
            raise ValueError("layout is not eligible for the fused halo path")
        self.geom = geom
        L = a.layout
        self.nyv = L.ny - 2 * L.nghost
        self.nzv = L.nz - 2 * L.nghost
        nc = a.ncomp
        shape = (L.nslots * nc, self.nzv, 2, self.nyv)
        self.xh = {id(a): torch.zeros(shape, dtype=torch.float64, device=a.device),
                   id(b): torch.zeros(shape, dtype=torch.float64, device=a.device)}
        table = face_neighbors(a, geom, multi)
        self.nbr = torch.as_tensor(table.reshape(-1), dtype=torch.int32, device=a.device)
        if max_rows is None:
            max_rows = default_fused_rows(a)
        self.plan = march_plan(a, True, max_rows, nctas)
        # Halo mode (include/tilemesh_b200.h): with columns of one height and 128-B aligned
        # rows the y/z halos are read from the neighbours' valid cells and the epilogue writes
        # only the packed x halos (FUSED_NBR); otherwise it also scatters y/z face ghosts of
        # the new field (FUSED_SCATTER).  Fixed for the lifetime of the pair.
        cols = self.plan.columns
        nbr_ok = len(set(cols["ny"].tolist())) == 1 and int(cols["nx"].max()) % 16 == 0
        self.mode = _native.HALO_FUSED_NBR if nbr_ok else _native.HALO_FUSED_SCATTER
        # Multi-rank: the column planes holding cells another rank needs (the source cells of the
        # halo exchange: remote faces, edges, corners) march first as one launch; they travel on a
        # side stream while every other plane marches as a second launch, so the NCCL exchange
        # overlaps the interior sweep even when every box touches another
        # rank (C2 strong-scaled: only its boundary planes / rows wait).  Each cell is still
        # computed exactly once, by the same kernel, so results do not change.
        self.plan_b = self.plan_i = None
        self.comm = None
        self.timeline = None  # a list: each multi-rank step appends its phase events
        if multi:
            cols = self.plan.columns
            # "boundary" slots: every slot whose cells travel to another rank (the source of
            # any send tag -- faces, edges and corners), not only slots with a remote face:
            # the exchange packs them on the comm stream while the interior columns march
            from .multifab import _device_fill
            from .fillplan import build_fill_plan as _bfp

            fp = fill_plan = fill_plan if fill_plan is not None else _bfp(a, geom)
            halo = _device_fill(a, fp)[1]
            bcols, icols = split_columns_by_sends(a, cols, halo.send_src if halo is not None else {})
            if len(bcols) and len(icols):
                self.plan_b = _native.MarchPlan(bcols, self.plan.nctas)
                self.plan_i = _native.MarchPlan(icols, self.plan.nctas)
                self.comm = torch.cuda.Stream(a.device)
        # faces whose neighbour is on another rank: filled by the halo exchange after each
        # step; x faces then copied from the ghost column into the packed x halo
        remote_x = [(s, side) for s in range(table.shape[0]) for side in (0, 1) if table[s, side] == REMOTE]
        # every rank joins the exchange (one collective per step), even one
        # whose faces all happen to be local
        self.remote = multi
        self.fill_plan = fill_plan
        if self.remote:
            every = [(s, side) for s in range(table.shape[0]) for side in (0, 1)]
            self._init_plan, self.xh_side = xh_own_ghost_plan(a, every, self.nyv, self.nzv)
            self._remote_x = xh_own_ghost_plan(a, remote_x, self.nyv, self.nzv)[0] if remote_x else None
        else:
            self._init_plan = self._xh_init_plan(a, table)

    def _xh_init_plan(self, mf: MultiFab, table) -> "_native.CopyPlan":
        plan, self.xh_side = xh_init_plan(mf, table, self.nyv, self.nzv)
        return plan

    def prime(self, mf: MultiFab, plan=None) -> None:
        """Fill every halo of ``mf`` from its valid data (regular FillBoundary
        + packed x halos)."""
        from .multifab import fill_boundary

        fill_boundary(mf, self.geom, plan)
        xh = self.xh[id(mf)]
        self._init_plan.run(xh.data_ptr(), self.xh_side, mf.ptr, mf.layout.side(), mf.stream())
        for p in (self.plan, self.plan_b, self.plan_i):
            if p is not None:
                _native.check(_native.load().tm_march_plan_reset_halos(p.handle), "tm_march_plan_reset_halos")

    def step(self, new: MultiFab, old: MultiFab, params, reverse: bool = False) -> None:
        """One fused step: sweep old -> new reading old's face halos and
        writing new's face halos (no separate FillBoundary).  ``reverse``
        walks the columns backwards (same results): alternating it between
        consecutive steps lets each step start on the planes the previous
        one wrote last, while they are still in L2."""
        import torch

        c = params.coefficients()

        def march(plan):
            _native.check(_native.load().tm_heat_march(
                plan.handle, old.layout.to_c(), old.ptr, new.wgptr, old.ncomp, c[0], c[1], c[2], c[3], self.mode,
                self.xh[id(old)].data_ptr(), self.xh[id(new)].data_ptr(), self.nbr.data_ptr(), int(reverse),
                old.stream()), "tm_heat_march(fused)")

        if not self.remote:
            march(self.plan)
            return
        # faces shared with other ranks: NCCL exchange of the new field's boundary
        from .fillplan import build_fill_plan
        from .multifab import _device_fill

        if self.fill_plan is None:
            self.fill_plan = build_fill_plan(new, self.geom)
        _, halo = _device_fill(new, self.fill_plan)

        def exchange():
            stream = new.stream()
            halo.start(new, stream)
            halo.finish(new, stream)
            if self._remote_x is not None:
                self._remote_x.run(self.xh[id(new)].data_ptr(), self.xh_side, new.ptr, new.layout.side(), stream)

        if self.comm is None:  # every local box touches another rank: nothing to overlap with
            march(self.plan)
            exchange()
            return
        main = torch.cuda.current_stream(new.device)
        tl = self.timeline  # optional: CUDA events marking the phases (tools/overlap_timeline.py)
        marks = None
        if tl is not None:
            marks = {k: torch.cuda.Event(enable_timing=True) for k in (
                "start", "boundary_done", "interior_start", "interior_done", "exchange_start", "exchange_done")}
            marks["start"].record(main)
        march(self.plan_b)
        boundary_done = torch.cuda.Event(enable_timing=tl is not None)
        boundary_done.record(main)
        # the interior columns are enqueued BEFORE the exchange: a host-blocking exchange (gloo)
        # then runs while they march, and an NCCL one on the side stream concurrently with them.
        # The exchange reads only the boundary planes' valid cells and writes only ghost cells of
        # remote faces (and their x halos); the interior march writes other cells
        if tl is not None:
            marks["interior_start"].record(main)
        march(self.plan_i)
        if tl is not None:
            marks["interior_done"].record(main)
        self.comm.wait_event(boundary_done)
        with torch.cuda.stream(self.comm):
            if tl is not None:
                marks["exchange_start"].record(self.comm)
            exchange()
            if tl is not None:
                marks["exchange_done"].record(self.comm)
        if tl is not None:
            marks["boundary_done"] = boundary_done
            tl.append(marks)
        main.wait_stream(self.comm)


class FusedGSRB:
    """Red-black Gauss-Seidel sweeps as two fused launches per sweep (red
    pass + halo scatter, black pass + halo scatter), in place on ``phi``.
    Bit-identical to ``stencil.gsrb_sweep`` (red, FillBoundary, black,
    FillBoundary)."""

    LONG = 8  # sweeps per replay of the long graph
    _long = None

    def __init__(self, phi: MultiFab, rhs: MultiFab, geom: Geometry, max_rows: int | None = None,
                 nctas: int | None = None):
        import torch

        if not fusable(phi, geom) or phi.ncomp != 1 or rhs.ncomp != 1:
            raise ValueError("layout is not eligible for the fused GSRB path")
        if phi.ba != rhs.ba or phi.local_units != rhs.local_units:
            raise ValueError("phi and rhs must share the BoxArray and distribution")
        self.phi, self.rhs, self.geom = phi, rhs, geom
        L = phi.layout
        self.nyv = L.ny - 2 * L.nghost
        self.nzv = L.nz - 2 * L.nghost
        self.xh = torch.zeros((L.nslots, self.nzv, 2, self.nyv), dtype=torch.float64, device=phi.device)
        table = face_neighbors(phi, geom)
        self.nbr = torch.as_tensor(table.reshape(-1), dtype=torch.int32, device=phi.device)
        self.plan = march_plan(phi, True, max_rows, nctas, rhs_rows=True)
        self._init, self.xh_side = xh_init_plan(phi, table, self.nyv, self.nzv)
        self.h2 = geom.dx[0] * geom.dx[0]
        self._graph = None

    def prime(self, plan=None) -> None:
        from .multifab import fill_boundary

        fill_boundary(self.phi, self.geom, plan)
        self._init.run(self.xh.data_ptr(), self.xh_side, self.phi.ptr, self.phi.layout.side(), self.phi.stream())

    def colour(self, color: int) -> None:
        phi, rhs = self.phi, self.rhs
        _native.check(_native.load().tm_gsrb_march(
            self.plan.handle, phi.layout.to_c(), phi.wgptr, rhs.layout.to_c(), rhs.ptr, color, self.h2,
            self.xh.data_ptr(), self.nbr.data_ptr(), phi.stream()), "tm_gsrb_march")

    def sweep(self) -> None:
        self.colour(0)
        self.colour(1)

    def run(self, sweeps: int, use_graph: bool = True) -> None:
        """``sweeps`` sweeps.  A colour pass is tens of microseconds of device
        time, less than the host cost of issuing it, so after one eager
        sweep (which also warms the plans) one sweep is captured as a CUDA
        graph and replayed."""
        import torch

        k = 0
        if use_graph and self._graph is None and sweeps >= 2:
            self.sweep()
            k = 1
            cur = torch.cuda.current_stream(self.phi.device)
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(self.phi.device)
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self.sweep()
            cur.wait_stream(s)
            self._graph = g
            # a second graph chaining LONG sweeps: every replay is a graph launch (~2 us)
            gl = torch.cuda.CUDAGraph()
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                with torch.cuda.graph(gl, stream=s):
                    for _ in range(self.LONG):
                        self.sweep()
            cur.wait_stream(s)
            self._long = gl
        if use_graph and getattr(self, "_long", None) is not None and self._graph is not None:
            while sweeps - k >= self.LONG:
                self._long.replay()
                k += self.LONG
        for _ in range(k, sweeps):
            if use_graph and self._graph is not None:
                self._graph.replay()
            else:
                self.sweep()

    def finalize(self, plan=None) -> None:
        from .multifab import fill_boundary

        fill_boundary(self.phi, self.geom, plan)


def split_eligible(phi: MultiFab, rhs: MultiFab, geom: Geometry) -> bool:
    """Colour-split GSRB: the fused layout rules, x extent a multiple of 4, and
    even periodic domain extents (a periodic image keeps its colour)."""
    if not fusable(phi, geom) or phi.ncomp != 1 or rhs.ncomp != 1 or phi.nghost != 1:
        return False
    if phi.ba != rhs.ba or phi.local_units != rhs.local_units:
        return False
    nx = phi.units[phi.local_units[0]].valid.extents[0]
    if nx % 4 or nx > 128:
        return False
    n = geom.domain.extents
    return all(n[d] % 2 == 0 for d in range(3) if geom.periodic[d])


class SplitGSRB:
    """GSRB sweeps on colour-split storage: ``prime`` splits phi (after a
    FillBoundary) and rhs into per-colour arrays, each colour pass is one
    launch reading only the other colour (and filling the face ghosts of its
    own), ``finalize`` merges back into phi and runs FillBoundary.
    Bit-identical to ``stencil.gsrb_sweep``."""

    LONG = FusedGSRB.LONG
    _long = None

    def __init__(self, phi: MultiFab, rhs: MultiFab, geom: Geometry, max_rows: int | None = None,
                 nctas: int | None = None):
        import torch

        if not split_eligible(phi, rhs, geom):
            raise ValueError("layout is not eligible for the colour-split GSRB path")
        self.phi, self.rhs, self.geom = phi, rhs, geom
        v = phi.units[phi.local_units[0]].valid
        self.nx, self.ny, self.nz = v.extents
        nh, n = self.nx // 2, len(phi.local_units)
        dev = phi.device
        self.c = [torch.zeros((n, self.nz + 2, self.ny + 2, nh + 8), dtype=torch.float64, device=dev)
                  for _ in range(2)]
        self.r = [torch.zeros((n, self.nz, self.ny, nh), dtype=torch.float64, device=dev) for _ in range(2)]
        par = [sum(phi.units[u].valid.lo) & 1 for u in phi.local_units]
        self.parity = torch.as_tensor(par, dtype=torch.int32, device=dev)
        self.nbr = torch.as_tensor(face_neighbors(phi, geom).reshape(-1), dtype=torch.int32, device=dev)
        # 32-row columns, one 17-warp CTA per SM: 48.9 us per C4 pass vs 50.5 for 16-row columns at
        # 2 CTAs per SM (r02, 8-stage ring)
        # (boxes wider than 64: 16-row columns keep the 8-stage ring inside shared memory)
        rows = max_rows or (32 if self.nx <= 64 else 16)
        self.plan = march_plan(phi, False, rows, nctas or (1 if rows > 16 else 2) * sm_count(dev),
                               tag="gsrb_split")
        self.h2 = geom.dx[0] * geom.dx[0]
        self._graph = None

    def prime(self, plan=None) -> None:
        from .multifab import fill_boundary

        phi, rhs = self.phi, self.rhs
        fill_boundary(phi, self.geom, plan)
        _native.check(_native.load().tm_gsrb_split(
            phi.layout.to_c(), phi.ptr, self.nx, self.ny, self.nz, self.parity.data_ptr(), self.c[0].data_ptr(),
            self.c[1].data_ptr(), rhs.layout.to_c(), rhs.ptr, self.r[0].data_ptr(), self.r[1].data_ptr(),
            phi.stream()), "tm_gsrb_split")

    def colour(self, color: int) -> None:
        _native.check(_native.load().tm_gsrb_split_pass(
            self.plan.handle, len(self.phi.local_units), self.nx, self.ny, self.nz, color, self.h2,
            self.c[1 - color].data_ptr(), self.c[color].data_ptr(), self.r[color].data_ptr(), self.nbr.data_ptr(),
            self.phi.stream()), "tm_gsrb_split_pass")

    def sweep(self) -> None:
        self.colour(0)
        self.colour(1)

    run = FusedGSRB.run

    def finalize(self, plan=None) -> None:
        from .multifab import fill_boundary

        phi = self.phi
        _native.check(_native.load().tm_gsrb_merge(
            phi.layout.to_c(), phi.wgptr, self.nx, self.ny, self.nz, self.parity.data_ptr(), self.c[0].data_ptr(),
            self.c[1].data_ptr(), phi.stream()), "tm_gsrb_merge")
        fill_boundary(phi, self.geom, plan)
