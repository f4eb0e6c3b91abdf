"""Stencil drivers: forward-Euler heat, red-black Gauss-Seidel, residual.

Reference: ``HeatParams`` (kernels.py:26-46), ``heat_step``
(kernels.py:174-215).  GSRB and the residual max-norm have no reference
(SURVEY.md §8a a12/a13); their canonical per-cell forms are fixed here and
in ``oracle/tm_oracle.c``.

Each driver validates on the host (``ValueError`` before any kernel runs,
as the reference does) and then issues ONE kernel launch covering every
tile of every box this rank owns, on the current torch stream.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

from . import _native
from .boxarray import Geometry
from .mfiter import TileSchedule, build_schedule
from .multifab import MultiFab, schedule_sweep_plan


@dataclass(frozen=True)
class HeatParams:
    diffusivity: float
    dt: float
    dx: tuple

    def __post_init__(self):
        if self.diffusivity <= 0 or self.dt <= 0 or any(d <= 0 for d in self.dx):
            raise ValueError("diffusivity, dt and dx must all be positive")

    @property
    def stability_limit(self) -> float:
        return 1.0 / (2.0 * self.diffusivity * sum(1.0 / d ** 2 for d in self.dx))

    @staticmethod
    def stable(diffusivity: float, dx, safety: float = 0.9) -> "HeatParams":
        """dt = safety x forward-Euler bound (same expression as the reference,
        so dt is bit-identical)."""
        if isinstance(dx, (int, float)):
            dx = (float(dx),) * 3
        limit = 1.0 / (2.0 * diffusivity * sum(1.0 / d ** 2 for d in dx))
        return HeatParams(diffusivity, safety * limit, tuple(dx))

    def coefficients(self) -> tuple:
        """(dxi0, dxi1, dxi2, dtD) computed as kernels.py:196-197 does."""
        dxi = tuple(1.0 / d for d in self.dx)
        return dxi + (self.diffusivity * self.dt,)


def _schedule_for(mf: MultiFab, schedule):
    if schedule is None:
        return build_schedule(mf, "off")
    if not isinstance(schedule, TileSchedule):
        return build_schedule(mf, schedule)
    return schedule


# Which kernel runs heat_step's sweep.  The tiling never changes a result
# (reference test_kernels.py:259-283), so large problems go to the persistent
# column march (Kernel A2 with x halos from the ghost columns: C2 61 us vs 64-68
# us for the tile kernel) and small ones, or zmerge requests, to the tile
# kernel.  "tiled" / "march" force one (tests).
SWEEP_KERNEL = "auto"
MARCH_MIN_CELLS = 1 << 21


def _use_march(mf: MultiFab, zmerge: bool) -> bool:
    from .march import march_eligible

    if SWEEP_KERNEL == "tiled" or zmerge:
        return False
    if not march_eligible(mf):
        if SWEEP_KERNEL == "march":
            raise ValueError("column march needs boxes of even x extent <= 128")
        return False
    if SWEEP_KERNEL == "march":
        return True
    big = mf._plans.get("march_big")
    if big is None:
        big = mf._plans["march_big"] = sum(mf.units[u].valid.ncells for u in mf.local_units) * mf.ncomp >= MARCH_MIN_CELLS
    return big


def heat_step(mf_new: MultiFab, mf_old: MultiFab, geom: Geometry, params: HeatParams,
              schedule: TileSchedule | None = None, workers: int = 1, arenas=None, verify: bool = False,
              zmerge: bool = False) -> None:
    """One forward-Euler step on every valid cell of every component; the
    ghosts of ``mf_old`` must have been filled (FillBoundary) beforehand.

    ``u_new`` is written on valid cells only; its ghosts are untouched
    (double buffering, reference kernels.py:4-7).  ``workers``/``arenas``
    are accepted for API parity: tile parallelism is the CTA grid and flux
    scratch lives in registers.  Unlike the reference (ncomp == 1 only,
    kernels.py:147-150) every component is updated, which is what config C3
    needs.
    """
    if mf_old.nghost < 1:
        raise ValueError("heat kernel requires nghost >= 1")
    if not mf_new.same_layout(mf_old):
        raise ValueError("mf_new and mf_old must share box layout, ncomp, nghost and distribution")
    if mf_new._data.data_ptr() == mf_old._data.data_ptr():
        raise ValueError("heat_step needs distinct old/new MultiFabs (double buffering)")
    if verify and params.dt > params.stability_limit:
        warnings.warn(f"dt={params.dt} exceeds stability bound {params.stability_limit}", stacklevel=2)
    if _use_march(mf_old, zmerge):
        from .march import heat_march

        heat_march(mf_new, mf_old, params, geom=geom)
        return
    sched = _schedule_for(mf_old, schedule)
    plan = schedule_sweep_plan(mf_old, sched, zmerge)
    if plan.nblocks == 0:
        return
    dxi0, dxi1, dxi2, dtD = params.coefficients()
    L = _native.load()
    _native.check(L.tm_heat_sweep(plan.handle, mf_old.layout.to_c(), mf_old.ptr, mf_new.wptr, 0, mf_old.ncomp,
                                  dxi0, dxi1, dxi2, dtD, mf_old.stream()), "tm_heat_sweep")


def _strides3(t, what: str):
    """(y, z) element strides of a device 3-D view with x contiguous."""
    if t.dim() < 3 or t.stride(0) != 1:
        raise ValueError(f"{what} must be a device array with x contiguous")
    return t.stride(1), t.stride(2)


def heat_flux(u, face_box, direction: int, dx: float, out=None):
    """F(face) = (u(high cell) - u(low cell)) / dx for every face in ``face_box``
    (reference kernels.py:86-120) on a device FAB; returns a device array shaped
    like the face box (x fastest, like the reference's F-order array)."""
    import torch

    from .box import Box

    if not face_box.itype[direction]:
        raise ValueError(f"face box must be node-centered in direction {direction}")
    cells = Box(tuple(lo - (1 if d == direction else 0) for d, lo in enumerate(face_box.lo)), face_box.hi)
    if not u.abox.contains(cells):
        raise ValueError(f"flux on {face_box} needs cells {cells}; fab only covers {u.abox}"
                         " (at least one filled ghost cell is required)")
    ex = face_box.extents
    view = u.data
    if out is None:
        out = torch.empty(tuple(reversed(ex)), dtype=torch.float64, device=view.device).permute(2, 1, 0)
    elif tuple(out.shape) != tuple(ex):
        raise ValueError(f"out has shape {tuple(out.shape)}, face box needs {tuple(ex)}")
    if any(e == 0 for e in ex):
        return out
    lo = u.abox.lo
    hi_cell = view[face_box.lo[0] - lo[0], face_box.lo[1] - lo[1], face_box.lo[2] - lo[2], 0]
    su = _strides3(view[..., 0], "u")
    so = _strides3(out, "out")
    _native.check(_native.load().tm_face_flux(hi_cell.data_ptr(), su[0], su[1], direction, ex[0], ex[1], ex[2],
                                              1.0 / dx, out.data_ptr(), so[0], so[1],
                                              _native.stream_handle(view.device)), "tm_face_flux")
    return out


def heat_divergence_update(u_new, u_old, fluxes, tile, params: HeatParams) -> None:
    """u_new = u_old + dt*D*div(F) on every cell of the tile (reference
    kernels.py:122-144); the flux arrays are indexed from tile.lo (heat_flux's
    output for the tile's three face boxes)."""
    fx, fy, fz = fluxes
    if u_new.abox.lo != u_old.abox.lo:
        raise ValueError("u_new and u_old must share an allocation box")
    e = tile.extents
    for f, d in ((fx, 0), (fy, 1), (fz, 2)):
        need = tuple(e[k] + (1 if k == d else 0) for k in range(3))
        if tuple(f.shape[:3]) != need:
            raise ValueError(f"flux {'xyz'[d]} has shape {tuple(f.shape)}, tile needs {need}")
    if any(v == 0 for v in e):
        return
    dxi = tuple(1.0 / d for d in params.dx)
    lo = u_old.abox.lo
    at = tuple(tile.lo[k] - lo[k] for k in range(3))
    vn, vo = u_new.data, u_old.data
    su = _strides3(vo[..., 0], "u_old")
    if _strides3(vn[..., 0], "u_new") != su:
        raise ValueError("u_new and u_old must have the same layout")
    sx, sy, sz = (_strides3(f, "flux") for f in fluxes)
    u_new._mf.wptr  # noqa: B018 -- a library kernel writes u_new's valid cells (state keys)
    _native.check(_native.load().tm_divergence_update(
        vn[at[0], at[1], at[2], 0].data_ptr(), vo[at[0], at[1], at[2], 0].data_ptr(), su[0], su[1],
        fx.data_ptr(), sx[0], sx[1], fy.data_ptr(), sy[0], sy[1], fz.data_ptr(), sz[0], sz[1], e[0], e[1], e[2],
        dxi[0], dxi[1], dxi[2], params.diffusivity * params.dt, _native.stream_handle(vo.device)),
        "tm_divergence_update")


def heat_sweep_plan(mf_new: MultiFab, mf_old: MultiFab, params: HeatParams, plan) -> None:
    """Kernel A over an explicit block table (e.g. the interior or boundary
    half of an overlapped step).  No checks: internal helper."""
    if plan.nblocks == 0:
        return
    dxi0, dxi1, dxi2, dtD = params.coefficients()
    _native.check(_native.load().tm_heat_sweep(plan.handle, mf_old.layout.to_c(), mf_old.ptr, mf_new.wptr, 0,
                                               mf_old.ncomp, dxi0, dxi1, dxi2, dtD, mf_old.stream()),
                  "tm_heat_sweep")


def overlapped_step(mf_new: MultiFab, mf_old: MultiFab, geom: Geometry, params: HeatParams, plan,
                    schedule: TileSchedule, zmerge: bool = False) -> None:
    """FillBoundary + heat sweep with the remote halo exchange overlapped:
    pack and post the NCCL sends/receives, run the intra-GPU copies and the
    sweep of every tile whose stencil cannot see a remote ghost, then wait
    for the messages, unpack and sweep the remaining (boundary) tiles.
    Results are identical to fill_boundary + heat_step."""
    from .multifab import _device_fill, overlap_sweep_plans

    copy, halo = _device_fill(mf_old, plan)
    stream = mf_old.stream()
    if halo is None:
        copy.run(mf_old.gptr, mf_old.layout.side(), mf_old.ptr, mf_old.layout.side(), stream)
        heat_step(mf_new, mf_old, geom, params, schedule, zmerge=zmerge)
        return
    inner, outer = overlap_sweep_plans(mf_old, schedule, halo.remote_dst, zmerge)
    halo.start(mf_old, stream)
    copy.run(mf_old.gptr, mf_old.layout.side(), mf_old.ptr, mf_old.layout.side(), stream)
    heat_sweep_plan(mf_new, mf_old, params, inner)
    halo.finish(mf_old, stream)
    heat_sweep_plan(mf_new, mf_old, params, outer)


def _check_poisson(phi: MultiFab, rhs: MultiFab):
    if phi.nghost < 1:
        raise ValueError("GSRB requires nghost >= 1 on phi")
    if phi.ncomp != 1 or rhs.ncomp != 1:
        raise ValueError("GSRB operates on single-component phi and rhs")
    if phi.ba != rhs.ba or phi.local_units != rhs.local_units:
        raise ValueError("phi and rhs must share the BoxArray and distribution")


def gsrb_color(phi: MultiFab, rhs: MultiFab, geom: Geometry, color: int,
               schedule: TileSchedule | None = None) -> None:
    """In-place red (0) or black (1) update ``phi = (sum6(phi) + h2*rhs)/6``
    on cells with ``(i+j+k)&1 == color``; h2 = dx*dx (cubic cells)."""
    _check_poisson(phi, rhs)
    if color not in (0, 1):
        raise ValueError("color must be 0 (red) or 1 (black)")
    h2 = geom.dx[0] * geom.dx[0]
    plan = schedule_sweep_plan(phi, _schedule_for(phi, schedule))
    if plan.nblocks == 0:
        return
    _native.check(_native.load().tm_gsrb_color(plan.handle, phi.layout.to_c(), phi.wgptr, rhs.layout.to_c(),
                                               rhs.ptr, color, h2, phi.stream()), "tm_gsrb_color")


def gsrb_sweep(phi: MultiFab, rhs: MultiFab, geom: Geometry, schedule=None, plan=None) -> None:
    """One sweep as BASELINE config 4 specifies: red, FillBoundary, black,
    FillBoundary."""
    from .multifab import fill_boundary

    gsrb_color(phi, rhs, geom, 0, schedule)
    fill_boundary(phi, geom, plan)
    gsrb_color(phi, rhs, geom, 1, schedule)
    fill_boundary(phi, geom, plan)


def residual_maxnorm(phi: MultiFab, rhs: MultiFab, geom: Geometry, schedule=None, device_out=None):
    """max over valid cells of ``|rhs + (sum6(phi) - 6 phi)/h2|``; ghosts of
    phi must be filled.  Returns a Python float (or writes ``device_out``)."""
    import torch

    _check_poisson(phi, rhs)
    h2 = geom.dx[0] * geom.dx[0]
    plan = schedule_sweep_plan(phi, _schedule_for(phi, schedule))
    out = device_out if device_out is not None else torch.zeros(1, dtype=torch.float64, device=phi.device)
    if plan.nblocks:
        _native.check(_native.load().tm_residual_maxnorm(plan.handle, phi.layout.to_c(), phi.ptr,
                                                         rhs.layout.to_c(), rhs.ptr, h2, out.data_ptr(),
                                                         phi.stream()), "tm_residual_maxnorm")
    from .multifab import comm_info

    if comm_info()[1] > 1:
        import torch.distributed as dist

        dist.all_reduce(out, op=dist.ReduceOp.MAX)
    if device_out is not None:
        return out
    return float(out.item())


def init_cosine(mf: MultiFab, geom: Geometry, modes=(1, 1, 1), offset: float = 0.0) -> None:
    """Valid data = offset + product of per-dimension cosines at cell
    centres: a discrete eigenfunction of the periodic 7-point operator
    (reference kernels.py:345-362)."""
    import numpy as np

    dom = geom.domain
    n = dom.extents

    def fn(i, j, k):
        return offset + (np.cos(2.0 * np.pi * modes[0] * (i - dom.lo[0] + 0.5) / n[0])
                         * np.cos(2.0 * np.pi * modes[1] * (j - dom.lo[1] + 0.5) / n[1])
                         * np.cos(2.0 * np.pi * modes[2] * (k - dom.lo[2] + 0.5) / n[2]))

    for c in range(mf.ncomp):
        mf.set_from_function(fn, c)


def heat_amplification(params: HeatParams, geom: Geometry, modes=(1, 1, 1)) -> float:
    """Exact per-step amplification of a cosine mode (kernels.py:365-377)."""
    import math

    n = geom.domain.extents
    g = 1.0
    for d in range(3):
        theta = 2.0 * math.pi * modes[d] / n[d]
        g += params.diffusivity * params.dt * (2.0 * math.cos(theta) - 2.0) / params.dx[d] ** 2
    return g


def gsrb_solve(phi: MultiFab, rhs: MultiFab, geom: Geometry, sweeps: int, schedule=None, plan=None,
               fused: bool | None = None, max_rows: int | None = None, split: bool | None = None) -> MultiFab:
    """``sweeps`` red-black sweeps (each: red, FillBoundary, black,
    FillBoundary -- BASELINE config 4).  With ``fused`` (default: whenever
    the layout allows) every colour pass is ONE launch that also scatters
    the updated colour into the neighbours' halos (march.FusedGSRB); with
    ``split`` (default: whenever eligible) the solve runs on colour-split
    storage, each pass reading only the other colour (march.SplitGSRB).  The
    result is bit-identical to the unfused loop and every ghost is filled
    on return."""
    from .march import FusedGSRB, SplitGSRB, fusable, split_eligible
    from .multifab import comm_info

    _check_poisson(phi, rhs)
    # caches key on the rhs LAYOUT, not its identity: a caller that builds a new rhs per solve
    # (multigrid, time loops) reuses one solver object, rebound to the new rhs below
    route_key = ("gsrb_route", geom, rhs.layout, tuple(rhs.local_units), comm_info()[1])
    route = phi._plans.get(route_key)
    if route is None:  # layout checks cost host time: once per (phi, rhs, geometry)
        can_ = comm_info()[1] == 1 and fusable(phi, geom)
        route = (can_, can_ and split_eligible(phi, rhs, geom))
        phi._plans[route_key] = route
    can, split_ok = route
    if fused and not can:
        raise ValueError("fused GSRB needs one rank and a uniform fully-covered box layout")
    if (can if fused is None else fused):
        use_split = split_ok if split is None else split
        key = ("fused_gsrb", geom, rhs.layout, tuple(rhs.local_units), max_rows, use_split)
        fg = phi._plans.get(key)
        if fg is None:
            fg = (SplitGSRB if use_split else FusedGSRB)(phi, rhs, geom, max_rows)
            phi._plans[key] = fg
        elif fg.rhs is not rhs:  # same layout, new array: rebind (the captured graph holds rhs pointers)
            fg.rhs = rhs
            fg._graph = fg._long = None
        fg.prime(plan)
        fg.run(sweeps)
        fg.finalize(plan)
        return phi
    for _ in range(sweeps):
        gsrb_sweep(phi, rhs, geom, schedule, plan)
    return phi
