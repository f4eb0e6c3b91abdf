"""Device-resident MultiFab and FillBoundary.

Reference: ``MultiFab`` (level.py:102-190), ``FArrayBox`` (fab.py:19-97),
``fill_boundary`` (level.py:297-323).

Storage (north star item 1): every MultiFab owns ONE
fp64 allocation of shape ``(nslots, ncomp, nz, ny, pitch)`` on its GPU, one
slot per unit this rank owns.  A unit's grown box sits at the slot origin
with its first valid cell at column ``xoff`` (a multiple of 16 doubles), so
every valid i-row starts on a 128-B boundary, and ``pitch`` is a multiple
of 16 doubles.  Within a slot the order is the reference's: x fastest, then
y, z, component slowest.  Uniform slots let one TMA tensor map describe the
whole MultiFab (dims x, y, z, slot*ncomp).

PyTorch is only the allocator here; every data-path operation is a kernel
of ``libtilemesh_b200.so`` launched on the current torch stream.
"""

from __future__ import annotations


import warnings
from typing import Callable, NamedTuple

import numpy as np

from . import _native
from .box import Box, check_tile_size, decompose, grow, split_extent
from .boxarray import BoxArray, DistributionMapping, Geometry
from .fab import BoxIndexed
from .fillplan import FillPlan, build_fill_plan
from .mfiter import TileSchedule, build_schedule

CONTIGUOUS = "contiguous"
REGIONAL = "regional"
ROW_ALIGN = 16  # doubles: 128 B
GHOST_ROW_WIDTH = 8  # doubles: one 64-B DRAM chunk per x-ghost row segment

# CTA tile limits of the sweep kernels (tm_stencil.cu): a block must fit the
# TMA box (nx + 2 <= 256) and at most 64 warp-row segments of 32 cells.
MAX_BLOCK_NX = 128
MAX_BLOCK_SEGS = 64


def _round_up(v: int, m: int) -> int:
    return -(-v // m) * m


def comm_info():
    """(rank, world_size) of the default torch.distributed group, or (0, 1)."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except ImportError:  # pragma: no cover
        pass
    return 0, 1


class StorageLayout(NamedTuple):
    nslots: int
    ncomp: int
    nghost: int
    pitch: int
    ny: int
    nz: int
    xoff: int

    @staticmethod
    def for_units(valids, ncomp: int, nghost: int) -> "StorageLayout":
        if valids:
            mx = max(v.extents[0] for v in valids)
            my = max(v.extents[1] for v in valids)
            mz = max(v.extents[2] for v in valids)
        else:
            mx = my = mz = 1
        xoff = _round_up(max(nghost, GHOST_ROW_WIDTH), ROW_ALIGN)
        # room for a full 64-B chunk on each side of the valid row (see local_copy_tags)
        pitch = _round_up(xoff + mx + max(nghost, GHOST_ROW_WIDTH), ROW_ALIGN)
        return StorageLayout(len(valids), ncomp, nghost, pitch, my + 2 * nghost, mz + 2 * nghost, xoff)

    @property
    def row(self) -> int:
        return self.pitch

    @property
    def plane(self) -> int:
        return self.pitch * self.ny

    @property
    def comp(self) -> int:
        return self.plane * self.nz

    @property
    def slot(self) -> int:
        return self.comp * self.ncomp

    def side(self) -> tuple:
        return (self.row, self.plane, self.comp)

    def to_c(self) -> "_native.tm_layout":
        return _native.tm_layout(*self)


def unit_boxes(ba, layout: str = CONTIGUOUS, region_size=None):
    """(unit valid boxes, owning grid per unit): one unit per grid
    (contiguous) or the grid's regions, ``decompose(grid, region_size)`` in
    grid order (regional, level.py:124-133).  Host-only."""
    valids, grid_of = [], []
    for g, grid in enumerate(ba):
        for v in ([grid] if layout == CONTIGUOUS else decompose(grid, check_tile_size(region_size))):
            valids.append(v)
            grid_of.append(g)
    return valids, grid_of


class Unit(NamedTuple):
    grid: int
    valid: Box
    fab: "DeviceFab | None"  # None for units owned by another rank


class DeviceFab(BoxIndexed):
    """One unit's FAB: a view of its slot in the MultiFab allocation.

    ``data`` is indexed like the reference's ``FArrayBox.data``:
    ``data[i - lo0, j - lo1, k - lo2, c]`` over the allocation (grown) box
    (a strided torch view, so writes land in the MultiFab).
    """

    def __init__(self, mf: "MultiFab", slot: int, abox: Box):
        self.abox = abox
        self.ncomp = mf.ncomp
        self.slot = slot
        self._mf = mf
        nx, ny, nz = abox.extents
        x0 = mf.layout.xoff - mf.nghost
        self._view = mf._data[slot, :, :nz, :ny, x0:x0 + nx].permute(3, 2, 1, 0)  # (x, y, z, c)

    @property
    def data(self):
        self._mf.settle()  # a deferred face fill is written before anyone sees the ghosts
        return self._view

    def at(self, i: int, j: int, k: int, c: int = 0) -> float:
        return float(self.data[self._local(i, j, k, c)].item())

    def set_at(self, i: int, j: int, k: int, v: float, c: int = 0) -> None:
        self.data[self._local(i, j, k, c)] = v

    def fill(self, v: float, region: Box | None = None, c: int | None = None) -> None:
        self.view(self.abox if region is None else region, 0 if c is None else c, None if c is None else 1).fill_(v)

    def to_numpy(self) -> np.ndarray:
        """Host copy in the reference layout: (nx, ny, nz, ncomp), F-order."""
        return np.asfortranarray(self.data.cpu().numpy())

    @property
    def flat(self) -> np.ndarray:
        """Host copy of the reference's flat storage (x fastest, component slowest)."""
        return self.to_numpy().ravel(order="F")


class MultiFab:
    """Device MultiFab with the reference constructor signature.

    ``dm`` (DistributionMapping over grids) selects the units this rank
    stores; by default grids are partitioned over the ranks of the default
    torch.distributed group (one rank when it is not initialised).
    """

    def __init__(self, ba: BoxArray, ncomp: int = 1, nghost: int = 0, layout: str = CONTIGUOUS,
                 region_size=None, zero: bool = True, dm: DistributionMapping | None = None,
                 device=None, rank: int | None = None):
        import torch

        if nghost < 0:
            raise ValueError(f"nghost must be non-negative, got {nghost}")
        if ncomp < 1:
            raise ValueError(f"ncomp must be positive, got {ncomp}")
        if layout not in (CONTIGUOUS, REGIONAL):
            raise ValueError(f"unknown layout {layout!r}")
        if layout == REGIONAL:
            if region_size is None:
                raise ValueError("regional layout requires a region_size")
            region_size = check_tile_size(region_size)
        if not torch.cuda.is_available():
            raise _native.TilemeshError("tilemesh_b200 MultiFab needs a CUDA device (no CPU fallback)")
        self.ba = ba
        self.ncomp = ncomp
        self.nghost = nghost
        self.layout_kind = layout
        self.region_size = region_size
        crank, cworld = comm_info()
        if dm is None:
            dm = DistributionMapping(ba, cworld)
        self.dm = dm
        self.rank = crank if rank is None else rank
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        valids, grid_of = unit_boxes(ba, layout, region_size)
        self.unit_owner = tuple(dm[g] for g in grid_of)  # a unit lives with its grid
        self.local_units = [u for u in range(len(valids)) if self.unit_owner[u] == self.rank]
        self.slot_of = {u: s for s, u in enumerate(self.local_units)}
        self.layout = StorageLayout.for_units([valids[u] for u in self.local_units], ncomp, nghost)
        L = self.layout
        shape = (L.nslots, ncomp, L.nz, L.ny, L.pitch)
        alloc = torch.zeros if zero else torch.empty
        self._data = alloc(shape, dtype=torch.float64, device=self.device)
        # Deferred ghosts of the reference-loop fast path (fill_boundary): y/z face ghosts the
        # next heat_step's sweep writes, and x face ghosts kept as a snapshot of the packed x
        # halos; written into storage ("settled") before anyone can observe them.
        self._pending_faces = None  # copy plan of the y/z face tags
        self._pending_edges = None  # copy plan of the edge/corner tags (run by the next sweep's fill warp)
        self._pending_cells = None  # ... and the same cells as a (dst, src) offset list for that warp
        self._w4_deferred = False   # the pending ghosts are a whole 4-deep fill (wide4 fast path)
        self._vx = None             # packed-halo snapshot holding the x face ghosts
        self._vx_nx = 0
        self._xh_spare = None       # second halo buffer: heat_step writes here while _xh is pinned
        self.settles = 0            # deferred ghosts written by copy launches (diagnostic)
        self.units = []
        for u, v in enumerate(valids):
            fab = None
            if u in self.slot_of:
                fab = DeviceFab(self, self.slot_of[u], grow(v, nghost) if nghost > 0 else v)
            self.units.append(Unit(grid_of[u], v, fab))
        self._plans: dict = {}
        self._unit_sweep = None
        self._scratch = {}
        # State keys of the reference-loop fast path (heat_step / fill_boundary):
        # ``valid_key`` changes whenever valid cells may have changed -- any torch in-place
        # write to ``data`` or a view of it (torch's version counter) or a library kernel
        # writing through ``wptr``; ``_xh_key`` is the valid_key for which the packed x
        # halos ``_xh`` hold the neighbours' boundary columns; ``_fill_key`` the valid_key
        # at the end of the last complete FillBoundary (ghosts consistent with valid data).
        self._writes = 0
        self._xh = None
        self._xh_key = None
        self._fill_key = None

    # ------------------------------------------------------------------ misc
    def clone_empty(self) -> "MultiFab":
        """Same layout and distribution, uninitialised storage (level.py:135-138)."""
        return MultiFab(self.ba, self.ncomp, self.nghost, self.layout_kind, self.region_size, zero=False,
                        dm=self.dm, device=self.device, rank=self.rank)

    def fab(self, u: int) -> DeviceFab:
        f = self.units[u].fab
        if f is None:
            raise KeyError(f"unit {u} is owned by rank {self.unit_owner[u]}, not {self.rank}")
        return f

    def __getitem__(self, mfi) -> DeviceFab:
        return self.fab(mfi.index() if hasattr(mfi, "index") else int(mfi))

    @property
    def data(self):
        """The storage tensor ``(nslots, ncomp, nz, ny, pitch)``.  Any pending face fill is
        written first, so every ghost a caller can observe is the reference's."""
        self.settle()
        return self._data

    def settle(self) -> None:
        """Write every deferred ghost (edges/corners and y/z faces: copy launches; x faces: one
        launch from the packed-halo snapshot) so the storage holds exactly a FillBoundary's
        ghosts."""
        if self._pending_faces is None and self._pending_edges is None and self._vx is None:
            return
        self.settles += 1
        self.settle_faces(count=False)
        if self._vx is not None:
            vx, self._vx = self._vx, None
            _native.check(_native.load().tm_xh_to_ghosts(self.layout.to_c(), self._data.data_ptr(), vx.data_ptr(),
                                                         self._vx_nx, _native.stream_handle(self.device)),
                          "tm_xh_to_ghosts")

    def settle_faces(self, count: bool = True) -> None:
        """Write pending edge/corner and y/z face ghosts (they are copied from valid cells:
        before those change)."""
        for name in ("_pending_edges", "_pending_faces"):
            pend = getattr(self, name)
            if pend is not None:
                setattr(self, name, None)
                self.settles += count
                pend.run(self._data.data_ptr(), self.layout.side(), self._data.data_ptr(), self.layout.side(),
                         _native.stream_handle(self.device))
        self._w4_deferred = False

    def drop_deferred(self) -> None:
        """A complete FillBoundary is about to rewrite every ghost the deferred ones cover."""
        self._pending_faces = None
        self._pending_edges = None
        self._w4_deferred = False
        self._vx = None

    @property
    def ptr(self) -> int:
        """Device address of the storage, for kernels that only READ it."""
        return self.data.data_ptr()

    @property
    def wptr(self) -> int:
        """Device address for a kernel that writes valid cells only (invalidates the
        packed x halos and the filled-ghost state).  Deferred x face ghosts stay
        deferred: their snapshot does not depend on the valid cells."""
        self.settle_faces()
        self._writes += 1
        return self._data.data_ptr()

    @property
    def wgptr(self) -> int:
        """Device address for a kernel that writes (or reads) ghost cells as well as
        valid ones: every deferred ghost is settled first."""
        self.settle()
        self._writes += 1
        return self._data.data_ptr()

    @property
    def gptr(self) -> int:
        """Device address for a kernel that writes ghost cells only (a fill or
        halo unpack; valid cells, and so the packed x halos, are unchanged)."""
        self._fill_key = None
        return self.data.data_ptr()

    def valid_key(self) -> tuple:
        return (self._data._version, self._writes)

    def xh_buffer(self):
        """Buffer a kernel writes this field's new packed x halos into:
        (slot*ncomp+c, nz, 2, ny) over valid y/z.  While the current buffer is
        pinned as the snapshot of deferred x face ghosts, the spare one."""
        import torch

        L = self.layout
        shape = (L.nslots * self.ncomp, L.nz - 2 * L.nghost, 2, L.ny - 2 * L.nghost)
        if self._xh is None:
            self._xh = torch.empty(shape, dtype=torch.float64, device=self.device)
        if self._vx is not None and self._vx is self._xh:
            if self._xh_spare is None:
                self._xh_spare = torch.empty(shape, dtype=torch.float64, device=self.device)
            self._xh, self._xh_spare = self._xh_spare, self._xh
        return self._xh

    def xh_current(self) -> bool:
        return self._xh is not None and self._xh_key == self.valid_key()

    def ghosts_current(self) -> bool:
        return self._fill_key is not None and self._fill_key == self.valid_key()

    def stream(self) -> int:
        return _native.stream_handle(self.device)

    def same_layout(self, other: "MultiFab") -> bool:
        return self.layout == other.layout and self.local_units == other.local_units and self.ba == other.ba

    # ----------------------------------------------------- host <-> device I/O
    def set_from_function(self, fn: Callable, comp: int = 0) -> None:
        """Valid cells of one component from ``fn(i, j, k)`` evaluated on the host."""
        import torch

        for u in self.local_units:
            v = self.units[u].valid
            I, J, K = np.ogrid[v.lo[0]:v.hi[0] + 1, v.lo[1]:v.hi[1] + 1, v.lo[2]:v.hi[2] + 1]
            vals = np.array(np.broadcast_to(np.asarray(fn(I, J, K), dtype=np.float64), v.extents), order="C")
            self.fab(u).view(v, comp, 1)[..., 0].copy_(torch.from_numpy(vals))

    def fill(self, v: float, comp: int | None = None) -> None:
        if comp is None:
            self.data.fill_(v)
        else:
            self.data[:, comp].fill_(v)

    def _global_copy_plan(self, domain: Box, direction: str):
        key = ("global", direction, domain)
        plan = self._plans.get(key)
        if plan is None:
            n = domain.extents
            gs = (n[0], n[0] * n[1], n[0] * n[1] * n[2])
            L = self.layout
            tags = np.zeros(len(self.local_units), dtype=_native.COPY_TAG_DTYPE)
            for t, u in enumerate(self.local_units):
                v = self.units[u].valid
                e = v.extents
                g_off = (v.lo[0] - domain.lo[0]) + gs[0] * (v.lo[1] - domain.lo[1]) + gs[1] * (v.lo[2] - domain.lo[2])
                m_off = self.slot_of[u] * L.slot + L.nghost * L.plane + L.nghost * L.row + L.xoff
                if direction == "scatter":
                    tags[t] = (m_off, g_off, e[0], e[1], e[2], 0)
                else:
                    tags[t] = (g_off, m_off, e[0], e[1], e[2], 0)
            plan = (_native.CopyPlan(tags, self.ncomp), gs)
            self._plans[key] = plan
        return plan

    def from_global(self, glob, domain: Box | None = None) -> None:
        """Valid cells from a domain-shaped array ``(ncomp, nz, ny, nx)``
        (numpy on the host, or a torch tensor on this device)."""
        import torch

        domain = self.ba_domain() if domain is None else domain
        if isinstance(glob, np.ndarray):
            g = torch.from_numpy(np.ascontiguousarray(glob, dtype=np.float64)).to(self.device, non_blocking=True)
        else:
            g = glob.to(self.device, dtype=torch.float64).contiguous()
        n = domain.extents
        if tuple(g.shape) != (self.ncomp, n[2], n[1], n[0]):
            raise ValueError(f"global array shape {tuple(g.shape)} != {(self.ncomp, n[2], n[1], n[0])}")
        plan, gs = self._global_copy_plan(domain, "scatter")
        plan.run(self.wptr, self.layout.side(), g.data_ptr(), gs, self.stream())
        self._keepalive = g

    def to_global(self, domain: Box | None = None, out=None):
        """Valid cells of the units this rank owns gathered into a device
        tensor ``(ncomp, nz, ny, nx)`` (cells of other ranks' units stay 0)."""
        import torch

        domain = self.ba_domain() if domain is None else domain
        n = domain.extents
        if out is None:
            out = torch.zeros((self.ncomp, n[2], n[1], n[0]), dtype=torch.float64, device=self.device)
        plan, gs = self._global_copy_plan(domain, "gather")
        plan.run(out.data_ptr(), gs, self.ptr, self.layout.side(), self.stream())
        return out

    def ba_domain(self) -> Box:
        from .box import bounding_box

        return bounding_box(self.ba)

    def grid_valid_array(self, g: int, comp: int = 0) -> np.ndarray:
        """Valid data of grid ``g`` as a host ``(nx, ny, nz)`` array (level.py:152-167)."""
        if self.layout_kind == CONTIGUOUS:
            u = self.units[g]
            return np.asfortranarray(self.fab(g).view(u.valid, comp, 1)[..., 0].cpu().numpy())
        grid = self.ba[g]
        out = np.empty(grid.extents, order="F")
        for u, unit in enumerate(self.units):
            if unit.grid != g:
                continue
            sl = tuple(slice(unit.valid.lo[d] - grid.lo[d], unit.valid.hi[d] - grid.lo[d] + 1) for d in range(3))
            out[sl] = self.fab(u).view(unit.valid, comp, 1)[..., 0].cpu().numpy()
        return out

    def _grid_shadow(self) -> "MultiFab":
        """Regional layout: a contiguous, ghost-free copy of the valid data (one
        slot per grid, same distribution), refreshed by one copy launch.  The
        reference checksum runs in grid order over whole grids, across region
        boundaries (level.py:183-190), which is the contiguous kernel's order."""
        sh = self._plans.get("grid_shadow")
        if sh is None:
            shadow = MultiFab(self.ba, self.ncomp, 0, dm=self.dm, device=self.device, rank=self.rank, zero=False)
            L, S = self.layout, shadow.layout
            tags = np.zeros(len(self.local_units), dtype=_native.COPY_TAG_DTYPE)
            for t, u in enumerate(self.local_units):
                unit = self.units[u]
                v, gb = unit.valid, self.ba[unit.grid]
                e = v.extents
                dst = (shadow.slot_of[unit.grid] * S.slot + (v.lo[2] - gb.lo[2]) * S.plane
                       + (v.lo[1] - gb.lo[1]) * S.row + S.xoff + (v.lo[0] - gb.lo[0]))
                src = self.slot_of[u] * L.slot + L.nghost * L.plane + L.nghost * L.row + L.xoff
                tags[t] = (dst, src, e[0], e[1], e[2], 0)
            sh = (shadow, _native.CopyPlan(tags, self.ncomp))
            self._plans["grid_shadow"] = sh
        shadow, plan = sh
        plan.run(shadow.wptr, shadow.layout.side(), self.ptr, self.layout.side(), self.stream())
        return shadow

    # -------------------------------------------------------------- reductions
    def _check_reduce(self, comp: int) -> None:
        if len(self.ba) == 0:
            raise ValueError("reduction over an empty BoxArray")
        if not 0 <= comp < self.ncomp:
            raise ValueError(f"component {comp} out of range")

    def unit_sweep_plan(self) -> "_native.SweepPlan":
        """One block per local unit covering its valid box, in unit order."""
        if self._unit_sweep is None:
            L = self.layout
            b = np.zeros(len(self.local_units), dtype=_native.BLOCK_DTYPE)
            for n, u in enumerate(self.local_units):
                v = self.units[u].valid
                e = v.extents
                b[n] = (self.slot_of[u], L.xoff, L.nghost, L.nghost, e[0], e[1], e[2], sum(v.lo) & 1)
            self._unit_sweep = _native.SweepPlan(b)
        return self._unit_sweep

    def _scratch_buf(self, name: str, n: int):
        import torch

        buf = self._scratch.get(name)
        if buf is None or buf.numel() < n:
            buf = torch.empty(max(n, 2), dtype=torch.float64, device=self.device)
            self._scratch[name] = buf
        return buf

    def reduce_sum_device(self, comp: int = 0):
        """Checksum on the device: a 1-element tensor, bit-identical to the
        reference ``reduce_sum`` (grid order, serial x-fastest per grid)."""
        import torch

        self._check_reduce(comp)
        if self.layout_kind == REGIONAL:
            return self._grid_shadow().reduce_sum_device(comp)
        rank, world = comm_info()
        nunits = len(self.units)
        L = _native.load()
        plan = self.unit_sweep_plan()
        if world == 1 or len(self.local_units) == nunits:
            part = self._scratch_buf("partial", max(nunits, 1))
            tot = self._scratch_buf("total", 2)
            _native.check(L.tm_reduce_sum(plan.handle, self.layout.to_c(), self.ptr, comp, part.data_ptr(),
                                          tot.data_ptr(), self.stream()), "tm_reduce_sum")
            return tot[:1]
        import torch.distributed as dist

        part = self._scratch_buf("partial", max(len(self.local_units), 1))
        tot = self._scratch_buf("total", 2)
        if self.local_units:
            _native.check(L.tm_reduce_sum(plan.handle, self.layout.to_c(), self.ptr, comp, part.data_ptr(),
                                          tot.data_ptr(), self.stream()), "tm_reduce_sum")
        full = torch.zeros(nunits, dtype=torch.float64, device=self.device)
        idx = torch.as_tensor(self.local_units, dtype=torch.long, device=self.device)
        full.index_copy_(0, idx, part[:len(self.local_units)])
        dist.all_reduce(full)  # each entry has exactly one non-zero contributor: exact
        # grid partials combined serially in grid order (nunits scalars)
        total = 0.0
        for v in full.cpu().tolist():
            total += v
        return torch.tensor([total], dtype=torch.float64, device=self.device)

    def reduce_sum(self, comp: int = 0) -> float:
        return float(self.reduce_sum_device(comp).item())

    def _minmax(self, comp: int):
        import torch

        self._check_reduce(comp)
        out = self._scratch_buf("minmax", 2)
        L = _native.load()
        rank, world = comm_info()
        if self.local_units:
            _native.check(L.tm_reduce_minmax(self.unit_sweep_plan().handle, self.layout.to_c(), self.ptr, comp,
                                             out.data_ptr(), self.stream()), "tm_reduce_minmax")
        else:
            out[0] = -float("inf")
            out[1] = float("inf")
        if world > 1:
            import torch.distributed as dist

            mx = out[:1].clone()
            mn = out[1:2].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(mn, op=dist.ReduceOp.MIN)
            return float(mx.item()), float(mn.item())
        o = out[:2].cpu()
        return float(o[0]), float(o[1])

    def reduce_max(self, comp: int = 0) -> float:
        return self._minmax(comp)[0]

    def reduce_min(self, comp: int = 0) -> float:
        return self._minmax(comp)[1]


def build_multifab(ba, ncomp=1, nghost=0, layout=CONTIGUOUS, region_size=None, **kw):
    return MultiFab(ba, ncomp, nghost, layout, region_size, **kw)


# --------------------------------------------------------------------------
# device tables
# --------------------------------------------------------------------------
def _tag_arrays(tags):
    n = len(tags)
    du = np.empty(n, dtype=np.int64)
    su = np.empty(n, dtype=np.int64)
    dlo = np.empty((n, 3), dtype=np.int64)
    slo = np.empty((n, 3), dtype=np.int64)
    ext = np.empty((n, 3), dtype=np.int64)
    for t, g in enumerate(tags):
        du[t] = g[0]
        su[t] = g[2]
        dlo[t] = g[1].lo
        slo[t] = g[3].lo
        ext[t] = g[1].extents
    return du, dlo, su, slo, ext


def cell_offsets(mf: MultiFab, units: np.ndarray, cells: np.ndarray) -> np.ndarray:
    """Element offsets in ``mf.data`` of global cells ``cells`` (n, 3) of
    units ``units`` (component 0)."""
    L = mf.layout
    tables = getattr(mf, "_unit_tables", None)
    if tables is None:  # per-MultiFab cache: valid lo corner and slot of every unit
        vlo = np.array([mf.units[u].valid.lo for u in range(len(mf.units))], dtype=np.int64).reshape(-1, 3)
        slot = np.full(len(mf.units), -1, dtype=np.int64)
        for u, sl in mf.slot_of.items():
            slot[u] = sl
        tables = (vlo, slot)
        try:
            mf._unit_tables = tables
        except AttributeError:
            pass
    vlo, slot = tables
    units = np.asarray(units, dtype=np.int64)
    cells = np.asarray(cells, dtype=np.int64).reshape(-1, 3)
    s = slot[units]
    if np.any(s < 0):
        raise ValueError("cell offsets requested for a unit this rank does not own")
    rel = cells - vlo[units]
    return (s * L.slot + (rel[:, 2] + L.nghost) * L.plane + (rel[:, 1] + L.nghost) * L.row
            + (rel[:, 0] + L.xoff))


def local_copy_tags(mf: MultiFab, tags) -> np.ndarray:
    """FillBoundary tags whose source and destination units both live on
    this rank, as device copy tags (both sides in ``mf.data``)."""
    if not tags:
        return np.zeros(0, dtype=_native.COPY_TAG_DTYPE)
    du, dlo, su, slo, ext = _tag_arrays(tags)
    out = np.zeros(len(tags), dtype=_native.COPY_TAG_DTYPE)
    out["dst_off"] = cell_offsets(mf, du, dlo)
    out["src_off"] = cell_offsets(mf, su, slo)
    out["ex"], out["ey"], out["ez"] = ext[:, 0], ext[:, 1], ext[:, 2]
    # x-face ghost rows: a tag that fills ALL ghost columns on one x side of
    # its rows copies a whole 64-B chunk instead of nghost isolated doubles:
    # the chunk holds those ghosts plus row padding that nothing reads, so the
    # write is a full DRAM chunk (no read-modify-write of a partial sector)
    # and the source read costs the same chunk it touched anyway.  Other tags
    # never write these rows' ghost columns (plan tags are disjoint in dst).
    ng, W = mf.nghost, GHOST_ROW_WIDTH
    if 0 < ng < W:
        vlo = np.array([mf.units[u].valid.lo[0] for u in range(len(mf.units))], dtype=np.int64)
        vhi = np.array([mf.units[u].valid.hi[0] for u in range(len(mf.units))], dtype=np.int64)
        full = ext[:, 0] == ng
        left = full & (dlo[:, 0] == vlo[du] - ng)
        right = full & (dlo[:, 0] == vhi[du] + 1)
        out["dst_off"][left] -= W - ng
        out["src_off"][left] -= W - ng
        out["ex"][left | right] = W
    return out


def _plan_key(mf: MultiFab):
    return (mf.layout, tuple(mf.local_units), mf.rank, mf.dm.nranks, mf.ncomp)


def _device_fill(mf: MultiFab, plan: FillPlan):
    key = _plan_key(mf)
    dev = plan._device.get(key)
    if dev is None:
        from .halo import HaloExchange

        owners = mf.unit_owner
        local = [t for t in plan.tags if owners[t.dst_unit] == mf.rank and owners[t.src_unit] == mf.rank]
        copy = _native.CopyPlan(local_copy_tags(mf, local), mf.ncomp)
        halo = HaloExchange(mf, plan) if mf.dm.nranks > 1 else None
        dev = (copy, halo)
        plan._device[key] = dev
    return dev


def fill_boundary(mf: MultiFab, geom: Geometry, plan: FillPlan | None = None, workers: int = 1) -> None:
    """Copy valid data into every fillable ghost cell (level.py:297-323).

    Intra-GPU tags run as one packed copy kernel; tags whose source box is
    on another rank travel as packed halo messages (``halo.HaloExchange``).
    ``workers`` is accepted for API parity and ignored (the kernel is the
    parallelism).
    """
    if plan is None:
        plan = mf._plans.get(("fill", geom))
        if plan is None:
            plan = build_fill_plan(mf, geom)
            mf._plans[("fill", geom)] = plan
    stream = mf.stream()
    fast = _xh_fill(mf, plan, geom) if mf.xh_current() else None
    w4 = _w4_fill(mf, plan, geom) if fast is None and mf.nghost == 4 else None
    if w4 is not None:
        # wide4 reference-loop fast path: every ghost is deferred; the next wide4_step writes the
        # face ghosts as it loads them from the neighbours and copies the edge/corner cells in the
        # same launch (tm_wide4_march_fill).  Anything observing or overwriting the field first
        # settles them (one copy launch each for faces and edges), as for heat_step's path.
        faces, edges, cells = w4
        mf.drop_deferred()
        mf._pending_faces, mf._pending_edges, mf._pending_cells = faces, edges, cells
        mf._w4_deferred = True
        mf._fill_key = mf.valid_key()
        return
    if fast is not None:
        # Reference-loop fast path.  The packed x halos the last heat_step wrote are current,
        # so the next heat_step can run the neighbour-halo march, whose y/z halo loads ARE this
        # fill's y/z face ghosts: it writes them as it goes (TM_HALO_FUSED_NBR_GHOSTS); the x face
        # ghosts ARE the packed halos, kept as a snapshot.  Here only the edge/corner tags run.
        # Deferred ghosts are written before anyone can observe them (MultiFab.data / .ptr /
        # FAB views / kernels that touch ghosts settle them), so no caller ever sees a ghost the
        # reference would not.
        edges, faces, nx, cells = fast
        mf.drop_deferred()
        mf._pending_faces = faces  # y/z faces: written by the next heat_step's sweep
        if cells is None:
            edges.run(mf.gptr, mf.layout.side(), mf.ptr, mf.layout.side(), stream)
        else:
            mf._pending_edges = edges  # edges/corners: copied by that sweep's fill warp (tm_heat_march_fill)
            mf._pending_cells = cells
        if _capturing() and not _SNAPSHOTS_IN_CAPTURE[0]:
            # a CUDA graph freezes buffer pointers, and pinning the halo buffer as a snapshot
            # makes the next heat_step write the other one: the pattern repeats only every two
            # steps per field.  Unknown captures get the x faces written now instead.
            _native.check(_native.load().tm_xh_to_ghosts(mf.layout.to_c(), mf._data.data_ptr(),
                                                         mf._xh.data_ptr(), nx, stream), "tm_xh_to_ghosts")
        else:
            mf._vx, mf._vx_nx = mf._xh, nx  # x faces: the packed halos of exactly this data
    else:
        mf.drop_deferred()
        copy, halo = _device_fill(mf, plan)
        if halo is not None:
            halo.start(mf, stream)
        copy.run(mf.gptr, mf.layout.side(), mf.ptr, mf.layout.side(), stream)
        if halo is not None:
            halo.finish(mf, stream)
    mf._fill_key = mf.valid_key()


FillBoundary = fill_boundary


_SNAPSHOTS_IN_CAPTURE = [False]


def _capturing() -> bool:
    import torch

    return torch.cuda.is_current_stream_capturing()


class snapshots_in_capture:
    """Context: the CUDA graph being captured replays a whole number of pairs of
    reference-loop steps per field (runner.HeatRunner's unfused 4-step graphs),
    so pinned packed-halo snapshots (fill_boundary's deferred x faces) repeat
    with the graph and may be used."""

    def __enter__(self):
        _SNAPSHOTS_IN_CAPTURE[0] = True
        return self

    def __exit__(self, *exc):
        _SNAPSHOTS_IN_CAPTURE[0] = False


def _xh_fill(mf: MultiFab, plan: FillPlan, geom: Geometry):
    """(copy plan of the edge/corner tags, copy plan of the y/z face tags, box width, the
    edge/corner cells as a device offset list or None) for a one-rank, one-ghost MultiFab on
    which heat_step runs the neighbour-halo march (the fast path of the reference loop), or
    None.  Cached per plan and layout."""
    key = ("xh_fill",) + _plan_key(mf)
    if key in plan._device:
        return plan._device[key]
    out = None
    from .march import xh_route

    route = xh_route(mf, geom) if mf.nghost == 1 and mf.dm.nranks == 1 else None
    L = mf.layout
    nx = mf.units[mf.local_units[0]].valid.extents[0] if mf.local_units else 0
    if route is not None and route[1] is not None and L.xoff >= 8 and L.xoff + nx + 8 <= L.pitch:
        edges, yz, xfaces = [], [], 0
        for t in plan.tags:
            v, d = mf.units[t.dst_unit].valid, t.dst_box
            out_dims = [k for k in range(3) if d.lo[k] < v.lo[k] or d.hi[k] > v.hi[k]]
            if len(out_dims) != 1:
                edges.append(t)
            elif out_dims[0] == 0:
                xfaces += d.ncells
            else:
                yz.append(t)
        # the x faces come from the packed halos, which hold one value per row and side of
        # every box: the plan must fill all of them (periodic / fully covered)
        ny, nz = mf.units[mf.local_units[0]].valid.extents[1:]
        if xfaces == 2 * ny * nz * len(mf.local_units):
            etags = local_copy_tags(mf, edges)
            out = (_native.CopyPlan(etags, mf.ncomp), _native.CopyPlan(local_copy_tags(mf, yz), mf.ncomp), nx,
                   _edge_cells(mf, etags))
    plan._device[key] = out
    return out


def _w4_fill(mf: MultiFab, plan: FillPlan, geom: Geometry):
    """(copy plan of the face tags, copy plan of the edge/corner tags, the edge/corner cells as
    a device offset list) for a one-rank MultiFab with exactly 4 ghost layers on which
    wide4_step can run Kernel W2 with neighbour-sourced halos (the wide4 reference loop's fast
    path), or None.  Cached per plan and layout."""
    key = ("w4_fill",) + _plan_key(mf)
    if key in plan._device:
        return plan._device[key]
    out = None
    if mf.nghost == 4 and mf.dm.nranks == 1 and mf.ncomp == 1 and mf.local_units:
        from .march import fusable
        from .wide4 import w2_nbr_eligible

        if fusable(mf, geom) and w2_nbr_eligible(mf):
            faces, edges = [], []
            for t in plan.tags:
                v, d = mf.units[t.dst_unit].valid, t.dst_box
                out_dims = [k for k in range(3) if d.lo[k] < v.lo[k] or d.hi[k] > v.hi[k]]
                (faces if len(out_dims) == 1 else edges).append(t)
            etags = local_copy_tags(mf, edges)
            cells = _edge_cells(mf, etags, chunk=4)
            if cells is not None:
                out = (_native.CopyPlan(local_copy_tags(mf, faces), mf.ncomp), _native.CopyPlan(etags, mf.ncomp),
                       cells)
    plan._device[key] = out
    return out


def _edge_cells(mf: MultiFab, tags, chunk: int = 1):
    """The edge/corner tags as a flat device list of (dst, src) element offsets, one pair per
    run of ``chunk`` cells along x (and component), for the fill warps of tm_heat_march_fill
    (chunk 1) / tm_wide4_march_fill (chunk 4: runs of 4 doubles, 32-B aligned) -- or None when a
    tag's x extent or offsets do not fit the chunk or the list would be large (> 64 MB)."""
    import torch

    L = mf.layout
    if any(int(t["ex"]) % chunk or int(t["dst_off"]) % chunk or int(t["src_off"]) % chunk for t in tags):
        return None
    n = int(sum(int(t["ex"]) * int(t["ey"]) * int(t["ez"]) for t in tags)) * mf.ncomp // chunk
    if n == 0 or 16 * n > 64 * 2 ** 20:
        return None
    rel = []
    for t in tags:
        x = np.arange(0, int(t["ex"]), chunk, dtype=np.int64)
        y = np.arange(int(t["ey"]), dtype=np.int64) * L.row
        z = np.arange(int(t["ez"]), dtype=np.int64) * L.plane
        c = np.arange(mf.ncomp, dtype=np.int64) * L.comp
        off = (c[:, None, None, None] + z[None, :, None, None] + y[None, None, :, None] + x).reshape(-1)
        rel.append(np.stack([off + int(t["dst_off"]), off + int(t["src_off"])], axis=1))
    cells = np.ascontiguousarray(np.concatenate(rel), dtype=np.int64)
    return torch.from_numpy(cells).to(mf.device)


# --------------------------------------------------------------------------
# sweep blocks from tile schedules
# --------------------------------------------------------------------------
def split_tile(tile: Box) -> list:
    """Cut a schedule tile into CTA-sized blocks (x <= 128, <= 64 row
    segments).  The stencil results do not depend on the cut."""
    e = tile.extents
    xs = split_extent(tile.lo[0], e[0], MAX_BLOCK_NX) if e[0] > MAX_BLOCK_NX else [(tile.lo[0], tile.hi[0])]
    out = []
    for (x0, x1) in xs:
        segs = -(-(x1 - x0 + 1) // 32)
        max_rows = max(1, MAX_BLOCK_SEGS // segs)
        ys = split_extent(tile.lo[1], e[1], max_rows) if e[1] > max_rows else [(tile.lo[1], tile.hi[1])]
        for (y0, y1) in ys:
            out.append(Box((x0, y0, tile.lo[2]), (x1, y1, tile.hi[2])))
    return out


def sweep_blocks(mf: MultiFab, entries, zmerge: bool = False) -> np.ndarray:
    """Device block table for (unit, tile) entries of this rank's units."""
    L = mf.layout
    rows = []
    for unit, tile in entries:
        if unit not in mf.slot_of:
            continue
        v = mf.units[unit].valid
        s = mf.slot_of[unit]
        for b in split_tile(tile):
            e = b.extents
            rows.append((s, L.xoff + b.lo[0] - v.lo[0], L.nghost + b.lo[1] - v.lo[1],
                         L.nghost + b.lo[2] - v.lo[2], e[0], e[1], e[2], (b.lo[0] + b.lo[1] + b.lo[2]) & 1))
    arr = np.array(rows, dtype=np.int64).reshape(-1, 8)
    if zmerge and len(arr):
        arr = merge_z(arr)
    out = np.zeros(len(arr), dtype=_native.BLOCK_DTYPE)
    for n, name in enumerate(_native.BLOCK_DTYPE.names):
        out[name] = arr[:, n]
    return out


def merge_z(arr: np.ndarray) -> np.ndarray:
    """Fuse blocks stacked in z over the same (slot, x, y) footprint into one
    longer k-march (bit-identical results, fewer halo planes re-read)."""
    order = np.lexsort((arr[:, 3], arr[:, 5], arr[:, 4], arr[:, 2], arr[:, 1], arr[:, 0]))
    a = arr[order]
    merged = []
    cur = a[0].copy()
    for r in a[1:]:
        if (r[0] == cur[0] and r[1] == cur[1] and r[2] == cur[2] and r[4] == cur[4] and r[5] == cur[5]
                and r[3] == cur[3] + cur[6]):
            cur[6] += r[6]
        else:
            merged.append(cur)
            cur = r.copy()
    merged.append(cur)
    return np.array(merged, dtype=np.int64)


def schedule_sweep_plan(mf: MultiFab, schedule: TileSchedule, zmerge: bool = False) -> "_native.SweepPlan":
    key = (mf.layout, tuple(mf.local_units), zmerge)
    plan = schedule._device.get(key)
    if plan is None:
        plan = _native.SweepPlan(sweep_blocks(mf, schedule.entries, zmerge))
        schedule._device[key] = plan
    return plan


def split_blocks(mf: MultiFab, blocks: np.ndarray, remote_dst: dict):
    """Split sweep blocks into (interior, boundary): a block is boundary when
    the 7-point stencil of one of its cells can touch a ghost cell that only
    a remote rank fills.  Interior blocks can run while the halo messages
    are in flight."""
    from .box import intersect as _isect

    L = mf.layout
    inner, outer = [], []
    for b in blocks:
        u = mf.local_units[int(b["slot"])]
        v = mf.units[u].valid
        lo = (v.lo[0] + int(b["x0"]) - L.xoff - 1, v.lo[1] + int(b["y0"]) - L.nghost - 1,
              v.lo[2] + int(b["z0"]) - L.nghost - 1)
        grown = Box(lo, (lo[0] + int(b["nx"]) + 1, lo[1] + int(b["ny"]) + 1, lo[2] + int(b["nz"]) + 1))
        hit = any(not _isect(grown, rb).is_empty for rb in remote_dst.get(u, ()))
        (outer if hit else inner).append(b)
    mk = lambda rows: np.array(rows, dtype=_native.BLOCK_DTYPE) if rows else np.zeros(0, dtype=_native.BLOCK_DTYPE)
    return mk(inner), mk(outer)


def overlap_sweep_plans(mf: MultiFab, schedule: TileSchedule, remote_dst: dict, zmerge: bool = False):
    """(interior, boundary) SweepPlans of a schedule for halo/compute overlap."""
    key = ("overlap", mf.layout, tuple(mf.local_units), zmerge, mf.rank, mf.dm.nranks)
    plans = schedule._device.get(key)
    if plans is None:
        inner, outer = split_blocks(mf, sweep_blocks(mf, schedule.entries, zmerge), remote_dst)
        plans = (_native.SweepPlan(inner), _native.SweepPlan(outer))
        schedule._device[key] = plans
    return plans
