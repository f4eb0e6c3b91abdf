"""The 9-point 8th-order Laplacian step ("wide4").

Reference: ``StencilCoeffs8`` / ``derive_coeffs8`` (kernels.py:49-83),
``wide4_step`` (kernels.py:218-247),
``wide4_amplification`` / ``wide4_stable_dt`` (kernels.py:380-404), cell form
``compiled.wide4_range`` (compiled.py:102-129).

Host code keeps the reference expressions (same dt, dxi2 and coefficient
bits); the update itself is ONE launch of Kernel W (``tm_wide4_march``,
csrc/tm_wide4.cu) over every box this rank owns, bit-identical to the
reference per cell.  It reuses the FillBoundary plan and kernel unchanged:
callers fill 4 ghost layers first, exactly as with the reference.

``Wide4Runner`` is the reference's step loop (fill_boundary; wide4_step)
on the device: with uniform boxes of at least 8^3 its steps are ONE launch
each, replayed from a CUDA graph of step pairs, and one regular FillBoundary
closes each ``advance``.  Boxes up to 64 wide run Kernel W2
(``tm_wide4_march_nbr``: 32-row columns, every 4-deep halo read from the face
neighbour's valid cells, nothing written but valid cells); wider boxes run
Kernel W with the face ghosts of the next step written by the epilogue
(``tm_wide4_march_fused``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .boxarray import Geometry
from .multifab import MultiFab

RADIUS = 4


@dataclass(frozen=True)
class StencilCoeffs8:
    """Centred second-derivative weights for offsets 0, +-1 .. +-4."""

    c0: float
    c1: float
    c2: float
    c3: float
    c4: float

    def as_array(self) -> np.ndarray:
        return np.array([self.c0, self.c1, self.c2, self.c3, self.c4])

    def weights9(self) -> np.ndarray:
        c = self.as_array()
        return np.array([c[4], c[3], c[2], c[1], c[0], c[1], c[2], c[3], c[4]])


def derive_coeffs8() -> StencilCoeffs8:
    """Even Taylor-moment system (weights sum 0, second moment 2, moments
    4, 6, 8 vanish) solved with ``numpy.linalg.solve`` as the reference does,
    so the coefficient bits are the reference's on the same host."""
    moments = [0, 2, 4, 6, 8]
    a = np.zeros((5, 5))
    rhs = np.zeros(5)
    for r, m in enumerate(moments):
        a[r, 0] = 1.0 if m == 0 else 0.0
        for n in range(1, 5):
            a[r, n] = 2.0 * n ** m
        if m == 2:
            rhs[r] = 2.0
    return StencilCoeffs8(*np.linalg.solve(a, rhs))


def wide4_amplification(diffusivity: float, dt: float, geom: Geometry, modes=(1, 1, 1),
                        coeffs: StencilCoeffs8 | None = None) -> float:
    """Per-step amplification of a cosine mode under the 9-point operator."""
    c = (coeffs if coeffs is not None else derive_coeffs8()).as_array()
    n = geom.domain.extents
    g = 1.0
    for d in range(3):
        theta = 2.0 * math.pi * modes[d] / n[d]
        s = c[0] + 2.0 * sum(c[k] * math.cos(k * theta) for k in range(1, 5))
        g += diffusivity * dt * s / geom.dx[d] ** 2
    return g


def wide4_stable_dt(diffusivity: float, dx, safety: float = 0.9) -> float:
    """dt at ``safety`` times the forward-Euler bound of the 9-point operator."""
    if isinstance(dx, (int, float)):
        dx = (float(dx),) * 3
    c = derive_coeffs8().as_array()
    s_pi = abs(c[0] + 2.0 * sum(c[k] * math.cos(k * math.pi) for k in range(1, 5)))
    lam = diffusivity * s_pi * sum(1.0 / d ** 2 for d in dx)
    return safety * 2.0 / lam


W2_ROWS = 32  # Kernel W2 column height cap (8 warps x 4 rows)


def _w2_rows(mf: MultiFab) -> int | None:
    """Column height cap under which every box of ``mf`` cuts into Kernel W2
    columns (width <= 64, even; row counts multiples of 4), else None."""
    from .march import _even_chunks

    exts = {mf.units[u].valid.extents for u in mf.local_units}
    for nx, ny, _ in exts:
        if nx > 64 or nx % 2 or ny % 2 or any(sz % 4 for _, sz in _even_chunks(ny, W2_ROWS)):
            return None
    return W2_ROWS if exts else None


def wide4_plan(mf: MultiFab, max_rows: int | None = None, nctas: int | None = None) -> "_native.MarchPlan":
    """Columns (full box width, full z) split into equal plane shares over one
    persistent CTA per SM: up to 32 rows when every box fits Kernel W2, else
    <= 16 rows (8 when wider than 64) for Kernel W."""
    from .march import march_columns, sm_count

    widest = max((mf.units[u].valid.extents[0] for u in mf.local_units), default=1)
    if widest > 128:
        raise ValueError("wide4 kernel supports boxes up to 128 cells wide in x")
    rows = max_rows or _w2_rows(mf) or (16 if widest <= 64 else 8)
    key = ("wide4", rows, nctas, mf.layout, tuple(mf.local_units))
    plan = mf._plans.get(key)
    if plan is None:
        cols = march_columns(mf, rows, packed=False)
        plan = _native.MarchPlan(cols, nctas or sm_count(mf.device))
        mf._plans[key] = plan
    return plan


def w2_nbr_eligible(mf: MultiFab) -> bool:
    """Uniform boxes that Kernel W2 runs with neighbour-sourced halos: width a multiple of 4
    (<= 64) and every box cut into columns of one height."""
    from .march import _even_chunks

    ext = {mf.units[u].valid.extents for u in mf.local_units}
    if len(ext) != 1 or _w2_rows(mf) is None:
        return False
    nx, ny, nz = next(iter(ext))
    return nx % 4 == 0 and min(nx, ny, nz) >= 2 * RADIUS and len({sz for _, sz in _even_chunks(ny, W2_ROWS)}) == 1


def _nbr_context(mf: MultiFab, geom: Geometry):
    """(device face-neighbour table, box extents) of a W2-NBR layout, cached per geometry."""
    import torch

    from .march import face_neighbors

    key = ("w4_nbr", geom)
    ctx = mf._plans.get(key)
    if ctx is None:
        nbr = torch.as_tensor(face_neighbors(mf, geom).reshape(-1), dtype=torch.int32, device=mf.device)
        box = (ctypes.c_int32 * 3)(*mf.units[mf.local_units[0]].valid.extents)
        ctx = (nbr, box)
        mf._plans[key] = ctx
    return ctx


def _launch_fill(mf_new: MultiFab, mf_old: MultiFab, geom: Geometry, diffusivity: float, dt: float,
                 coeffs: StencilCoeffs8 | None) -> None:
    """The wide4 step of the reference loop's fast path: the deferred fill of mf_old and the
    step in one launch (tm_wide4_march_fill)."""
    c = coeffs if coeffs is not None else derive_coeffs8()
    dxi2 = tuple(1.0 / d ** 2 for d in geom.dx)
    plan = wide4_plan(mf_old)
    nbr, box = _nbr_context(mf_old, geom)
    cells = mf_old._pending_cells
    cbuf = (ctypes.c_double * 5)(c.c0, c.c1, c.c2, c.c3, c.c4)
    new_ptr = mf_new.wptr
    _native.check(_native.load().tm_wide4_march_fill(
        plan.handle, mf_old.layout.to_c(), mf_old._data.data_ptr(), new_ptr, 1, ctypes.cast(cbuf, ctypes.c_void_p),
        dxi2[0], dxi2[1], dxi2[2], diffusivity * dt, nbr.data_ptr(), box, cells.data_ptr(), cells.shape[0],
        mf_old.stream()), "tm_wide4_march_fill")
    mf_old._pending_faces = mf_old._pending_edges = mf_old._pending_cells = None
    mf_old._w4_deferred = False


def _check(mf_new: MultiFab, mf_old: MultiFab) -> None:
    if mf_new.ncomp != 1 or mf_old.ncomp != 1:
        raise ValueError("stencil kernels operate on single-component MultiFabs")
    if mf_old.nghost < RADIUS:
        raise ValueError("wide4 kernel requires nghost >= 4")
    if not mf_new.same_layout(mf_old):
        raise ValueError("mf_new and mf_old must share box layout, ncomp, nghost and distribution")
    if mf_new._data.data_ptr() == mf_old._data.data_ptr():  # (not .data: that settles deferred ghosts)
        raise ValueError("wide4_step needs distinct old/new MultiFabs (double buffering)")


def _launch(mf_new: MultiFab, mf_old: MultiFab, geom: Geometry, diffusivity: float, dt: float,
            coeffs: StencilCoeffs8 | None, max_rows: int | None = None, nctas: int | None = None) -> None:
    c = coeffs if coeffs is not None else derive_coeffs8()
    dxi2 = tuple(1.0 / d ** 2 for d in geom.dx)
    dtD = diffusivity * dt
    plan = wide4_plan(mf_old, max_rows, nctas)
    if plan.ncolumns == 0:
        return
    cbuf = (ctypes.c_double * 5)(c.c0, c.c1, c.c2, c.c3, c.c4)
    _native.check(_native.load().tm_wide4_march(plan.handle, mf_old.layout.to_c(), mf_old.ptr, mf_new.wptr, 1,
                                                ctypes.cast(cbuf, ctypes.c_void_p), dxi2[0], dxi2[1], dxi2[2],
                                                dtD, mf_old.stream()), "tm_wide4_march")


def wide4_step(mf_new: MultiFab, mf_old: MultiFab, geom: Geometry, diffusivity: float, dt: float,
               schedule=None, workers: int = 1, coeffs: StencilCoeffs8 | None = None) -> None:
    """u_new = u_old + dt*D*(8th-order Laplacian) on every valid cell; the 4
    ghost layers of ``mf_old`` must be filled beforehand.  ``schedule`` and
    ``workers`` are accepted for API parity (the result does not depend on
    the tiling, reference test_kernels.py:360-368): the device
    decomposition is the persistent column march."""
    _check(mf_new, mf_old)
    if mf_old._w4_deferred and mf_old._pending_faces is not None:
        _launch_fill(mf_new, mf_old, geom, diffusivity, dt, coeffs)  # the fill rides on this launch
        return
    _launch(mf_new, mf_old, geom, diffusivity, dt, coeffs)


class Wide4Runner:
    """Owns an old/new pair and advances the wide4 diffusion ``n`` steps at a
    time; bit-identical to ``steps x (fill_boundary; wide4_step)``.  Fused
    (default when eligible): one launch per step -- with ``nbr_halos`` (default
    when the boxes allow Kernel W2) every halo is read from the face
    neighbours' valid cells and no ghost is written; otherwise the previous
    step's epilogue writes the face ghosts (Kernel W, scatter).  Unfused:
    FillBoundary + Kernel W/W2 per step."""

    LONG_PAIRS = 8  # captured pairs per replay of the long graph
    _long = None

    def __init__(self, mf: MultiFab, geom: Geometry, diffusivity: float, dt: float,
                 coeffs: StencilCoeffs8 | None = None, fused: bool | None = None,
                 use_graph: bool | None = None, nbr_halos: bool | None = None):
        import torch

        from .march import face_neighbors, fusable
        from .multifab import comm_info

        if mf.nghost < RADIUS or mf.ncomp != 1:
            raise ValueError("wide4 runner needs a single-component MultiFab with nghost >= 4")
        self.geom, self.diffusivity, self.dt = geom, diffusivity, dt
        self.coeffs = coeffs if coeffs is not None else derive_coeffs8()
        self.a = mf
        self.b = mf.clone_empty()
        world = comm_info()[1]
        ext = {mf.units[u].valid.extents for u in mf.local_units}
        can_fuse = (world == 1 and fusable(mf, geom) and len(ext) == 1 and min(next(iter(ext))) >= 2 * RADIUS)
        if fused and not can_fuse:
            raise ValueError("fused wide4 needs one rank and uniform boxes of at least 8^3 covering the domain")
        self.fused = can_fuse if fused is None else fused
        self.use_graph = (world == 1) if use_graph is None else (use_graph and world == 1)
        self.nbr_halos = False
        if self.fused:
            self.nbr = torch.as_tensor(face_neighbors(mf, geom).reshape(-1), dtype=torch.int32, device=mf.device)
            self.box = (ctypes.c_int32 * 3)(*next(iter(ext)))
            from .march import _even_chunks

            nx, ny, _ = next(iter(ext))
            # Kernel W2 with neighbour-sourced halos (no ghost writes at all): widths a multiple
            # of 4, every box cut into columns of one height
            can_nbr = (_w2_rows(mf) is not None and nx % 4 == 0
                       and len({sz for _, sz in _even_chunks(ny, W2_ROWS)}) == 1)
            if nbr_halos and not can_nbr:
                raise ValueError("neighbour-sourced wide4 halos need box widths that are multiples of 4 (<= 64) "
                                 "and box heights that cut into equal 4-row-multiple columns")
            self.nbr_halos = can_nbr if nbr_halos is None else nbr_halos
        self._graph = None
        self._primed = False
        self.steps_done = 0

    @property
    def current(self) -> MultiFab:
        return self.a if self.steps_done % 2 == 0 else self.b

    def reset(self) -> None:
        """Call after modifying ``a`` from outside: restart at step 0."""
        self.steps_done = 0
        self._primed = False

    def close(self) -> None:
        self._graph = self._long = None

    def _step(self, old: MultiFab, new: MultiFab) -> None:
        from .multifab import fill_boundary

        if not self.fused:
            fill_boundary(old, self.geom)
            wide4_step(new, old, self.geom, self.diffusivity, self.dt, coeffs=self.coeffs)
            return
        c = self.coeffs
        dxi2 = tuple(1.0 / d ** 2 for d in self.geom.dx)
        cbuf = (ctypes.c_double * 5)(c.c0, c.c1, c.c2, c.c3, c.c4)
        if self.nbr_halos:
            plan = wide4_plan(old)
            _native.check(_native.load().tm_wide4_march_nbr(
                plan.handle, old.layout.to_c(), old.ptr, new.wptr, 1, ctypes.cast(cbuf, ctypes.c_void_p),
                dxi2[0], dxi2[1], dxi2[2], self.diffusivity * self.dt, self.nbr.data_ptr(), self.box,
                old.stream()), "tm_wide4_march_nbr")
            return
        plan = wide4_plan(old, 16 if old.units[old.local_units[0]].valid.extents[0] <= 64 else 8)
        _native.check(_native.load().tm_wide4_march_fused(
            plan.handle, old.layout.to_c(), old.ptr, new.wgptr, 1, ctypes.cast(cbuf, ctypes.c_void_p),
            dxi2[0], dxi2[1], dxi2[2], self.diffusivity * self.dt, self.nbr.data_ptr(), self.box, old.stream()),
            "tm_wide4_march_fused")

    def _capture(self) -> None:
        import torch

        self._step(self.a, self.b)  # warm plans and tensor maps outside capture
        self._step(self.b, self.a)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            self._step(self.a, self.b)
            self._step(self.b, self.a)
        torch.cuda.current_stream().wait_stream(s)
        self._graph = g
        gl = torch.cuda.CUDAGraph()  # LONG_PAIRS pairs per replay: one graph launch per 16 steps
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(gl, stream=s):
            for _ in range(self.LONG_PAIRS):
                self._step(self.a, self.b)
                self._step(self.b, self.a)
        torch.cuda.current_stream().wait_stream(s)
        self._long = gl

    def advance(self, n: int, finalize: bool = True) -> MultiFab:
        """Advance ``n`` steps; returns the MultiFab holding the state (all
        ghosts filled when ``finalize``)."""
        from .multifab import fill_boundary

        if self.fused and not self._primed:
            fill_boundary(self.current, self.geom)
            self._primed = True
        k = 0
        if self.use_graph and self.steps_done % 2 == 0 and n >= 2:
            if self._graph is None:
                self._capture()  # two real steps
                self.steps_done += 2
                k += 2
            while n - k >= 2 * self.LONG_PAIRS:
                self._long.replay()
                self.steps_done += 2 * self.LONG_PAIRS
                k += 2 * self.LONG_PAIRS
            while n - k >= 2:
                self._graph.replay()
                self.steps_done += 2
                k += 2
        while k < n:
            old, new = (self.a, self.b) if self.steps_done % 2 == 0 else (self.b, self.a)
            self._step(old, new)
            self.steps_done += 1
            k += 1
        if finalize:
            fill_boundary(self.current, self.geom)
        return self.current
