"""CPU oracle for the stencil-sweep + FillBoundary path.

TEST INFRASTRUCTURE ONLY.  Imported by ``tests/``, ``__graft_entry__.smoke``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- as the
checker and as the CPU baseline, never as the product path.  The package
``paper_1604_03570_b200`` must not import this module.

Two independent restatements of the reference
(``/root/reference/pkg/src/tilemesh``):

1. ``HostMF`` + ``liboracle.so`` (``tm_oracle.c``): per-unit FABs laid out
   like the reference ``FArrayBox`` (fab.py:19-42), copy tags applied as
   ``_run_tags`` does (level.py:290-294), the four-loop tiled heat kernel
   of ``compiled.heat_tiles`` (compiled.py:32-99), ``serial_sum`` /
   ``reduce_sum`` (compiled.py:20-29, level.py:183-190), and the
   builder-owned GSRB / residual forms (no reference: parity unpinned).
2. ``heat_periodic``: whole-domain numpy form (``np.pad(mode="wrap")`` +
   the same per-cell arithmetic), SURVEY.md §8c's oracle for configs too
   big for a per-box plan.

``ref_fill_tags`` restates the reference's O(n^2) ``build_fill_plan``
(level.py:240-287) literally, to pin the O(n) planner on small layouts.

Pinning: ``tests/test_oracle.py`` checks all of the above against
``tests/golden/*.npz``, produced by ``tests/golden/make_golden.py`` from the
reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from math import ceil

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def lib():
    """Load (building on first use) ``oracle/liboracle.so``."""
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        src = os.path.join(HERE, "tm_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = ctypes.CDLL(path)
        L.orc_fill_tags.argtypes = [_f64p, _i64p, _i64p, _i64p, ctypes.c_int, _i64p, ctypes.c_int64, ctypes.c_int]
        L.orc_fill_tags.restype = None
        L.orc_heat_tiles.argtypes = [_f64p, _f64p, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_int]
        L.orc_heat_tiles.restype = None
        L.orc_wide4_tiles.argtypes = [_f64p, _f64p, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64] + \
            [ctypes.c_double] * 9 + [ctypes.c_int]
        L.orc_wide4_tiles.restype = None
        L.orc_serial_sum.argtypes = [_f64p, _i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int, _i64p, _i64p]
        L.orc_serial_sum.restype = ctypes.c_double
        L.orc_reduce_sum.argtypes = [_f64p, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int]
        L.orc_reduce_sum.restype = ctypes.c_double
        L.orc_gsrb_color.argtypes = [_f64p, _i64p, _i64p, _i64p, _f64p, _i64p, _i64p, _i64p, _i64p,
                                     ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_int]
        L.orc_gsrb_color.restype = None
        L.orc_residual_max.argtypes = [_f64p, _i64p, _i64p, _i64p, _f64p, _i64p, _i64p, _i64p, _i64p,
                                       ctypes.c_int64, ctypes.c_double, ctypes.c_int]
        L.orc_residual_max.restype = ctypes.c_double
        L.orc_max_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(t)


def max_threads() -> int:
    return int(lib().orc_max_threads())


# --------------------------------------------------------------------------
# Host MultiFab (reference FArrayBox layout)
# --------------------------------------------------------------------------
class HostMF:
    """Units = valid boxes (tuples lo, hi); FAB = grown box, F-order
    ``(nx, ny, nz, ncomp)``, all units in one flat buffer."""

    def __init__(self, valids, ncomp: int, nghost: int, fill: float = 0.0):
        self.valids = [(tuple(v.lo), tuple(v.hi)) if hasattr(v, "lo") else (tuple(v[0]), tuple(v[1]))
                       for v in valids]
        self.ncomp = ncomp
        self.nghost = nghost
        n = len(self.valids)
        self.lo = np.array([[l - nghost for l in v[0]] for v in self.valids], dtype=np.int64).reshape(n, 3)
        hi = np.array([[h + nghost for h in v[1]] for v in self.valids], dtype=np.int64).reshape(n, 3)
        self.ext = hi - self.lo + 1
        sizes = self.ext.prod(axis=1) * ncomp
        self.off = np.zeros(n, dtype=np.int64)
        if n:
            self.off[1:] = np.cumsum(sizes)[:-1]
        self.buf = np.full(int(sizes.sum()), fill, dtype=np.float64)
        self.valid_tab = np.array([list(v[0]) + list(v[1]) for v in self.valids], dtype=np.int64).reshape(n, 6)

    def fab(self, u: int) -> np.ndarray:
        e = self.ext[u]
        a = self.off[u]
        return self.buf[a:a + int(e.prod()) * self.ncomp].reshape(tuple(e) + (self.ncomp,), order="F")

    def valid_view(self, u: int, comp: int = 0) -> np.ndarray:
        g = self.nghost
        e = self.ext[u]
        return self.fab(u)[g:e[0] - g, g:e[1] - g, g:e[2] - g, comp]

    def from_global(self, glob: np.ndarray, dom_lo=(0, 0, 0)) -> None:
        """Valid cells from a global ``(ncomp, nz, ny, nx)`` array."""
        for u, (lo, hi) in enumerate(self.valids):
            sl = tuple(slice(lo[d] - dom_lo[d], hi[d] - dom_lo[d] + 1) for d in (2, 1, 0))
            for c in range(self.ncomp):
                self.valid_view(u, c)[...] = glob[(c,) + sl].transpose(2, 1, 0)

    def to_global(self, shape, dom_lo=(0, 0, 0)) -> np.ndarray:
        out = np.zeros((self.ncomp,) + tuple(shape))
        for u, (lo, hi) in enumerate(self.valids):
            sl = tuple(slice(lo[d] - dom_lo[d], hi[d] - dom_lo[d] + 1) for d in (2, 1, 0))
            for c in range(self.ncomp):
                out[(c,) + sl] = self.valid_view(u, c).transpose(2, 1, 0)
        return out

    def tables(self):
        return (np.ascontiguousarray(self.off), np.ascontiguousarray(self.lo.reshape(-1)),
                np.ascontiguousarray(self.ext.reshape(-1)))


def tags_array(tags) -> np.ndarray:
    """CopyTag-likes -> (n, 11) int64 rows: du, dlo, dhi, su, slo."""
    arr = np.empty((len(tags), 11), dtype=np.int64)
    for n, t in enumerate(tags):
        arr[n, 0] = t[0]
        arr[n, 1:4] = t[1].lo
        arr[n, 4:7] = t[1].hi
        arr[n, 7] = t[2]
        arr[n, 8:11] = t[3].lo
    return arr


def tiles_array(tiles) -> np.ndarray:
    """(unit, Box) pairs -> (n, 7) int64 rows: unit, lo, hi."""
    arr = np.empty((len(tiles), 7), dtype=np.int64)
    for n, (u, b) in enumerate(tiles):
        arr[n, 0] = u
        arr[n, 1:4] = b.lo
        arr[n, 4:7] = b.hi
    return arr


def fill_boundary(mf: HostMF, tags, nthreads: int = 1) -> None:
    arr = tags if isinstance(tags, np.ndarray) else tags_array(tags)
    arr = np.ascontiguousarray(arr, dtype=np.int64)
    off, lo, ext = mf.tables()
    lib().orc_fill_tags(_p(mf.buf, _f64p), _p(off, _i64p), _p(lo, _i64p), _p(ext, _i64p), mf.ncomp,
                        _p(arr, _i64p), len(arr), nthreads)


def heat_step(new: HostMF, old: HostMF, tiles, dxi, dtD: float, nthreads: int = 1) -> None:
    """Reference kernels.heat_step per component (C3 drives heat_tiles per
    component because heat_step rejects ncomp != 1: kernels.py:147-150)."""
    arr = tiles if isinstance(tiles, np.ndarray) else tiles_array(tiles)
    arr = np.ascontiguousarray(arr, dtype=np.int64)
    off, lo, ext = old.tables()
    for c in range(old.ncomp):
        lib().orc_heat_tiles(_p(new.buf, _f64p), _p(old.buf, _f64p), _p(off, _i64p), _p(lo, _i64p),
                             _p(ext, _i64p), _p(arr, _i64p), len(arr), c, dxi[0], dxi[1], dxi[2], dtD,
                             nthreads)


def wide4_step(new: HostMF, old: HostMF, tiles, coeffs, dxi2, dtD: float, nthreads: int = 1) -> None:
    """Reference kernels.wide4_step (kernels.py:218-247) over ``tiles`` of
    component 0, cell form compiled.wide4_range (compiled.py:102-129)."""
    arr = tiles if isinstance(tiles, np.ndarray) else tiles_array(tiles)
    arr = np.ascontiguousarray(arr, dtype=np.int64)
    off, lo, ext = old.tables()
    c = [float(v) for v in coeffs]
    lib().orc_wide4_tiles(_p(new.buf, _f64p), _p(old.buf, _f64p), _p(off, _i64p), _p(lo, _i64p), _p(ext, _i64p),
                          _p(arr, _i64p), len(arr), c[0], c[1], c[2], c[3], c[4], dxi2[0], dxi2[1], dxi2[2], dtD,
                          nthreads)


def wide4_periodic(u: np.ndarray, steps: int, coeffs, dxi2, dtD: float) -> np.ndarray:
    """Whole-domain numpy form, fully periodic; ``u`` (nz, ny, nx)."""
    c = [float(v) for v in coeffs]
    u = np.array(u, dtype=np.float64, copy=True)
    for _ in range(steps):
        p = np.pad(u, 4, mode="wrap")
        n = u.shape
        core = p[4:4 + n[0], 4:4 + n[1], 4:4 + n[2]]

        def sh(axis, m):
            sl = [slice(4, 4 + n[0]), slice(4, 4 + n[1]), slice(4, 4 + n[2])]
            sl[axis] = slice(4 + m, 4 + m + n[axis])
            return p[tuple(sl)]

        s = []
        for axis in (2, 1, 0):  # x, y, z
            acc = c[0] * core
            for m in range(1, 5):
                acc = acc + c[m] * (sh(axis, -m) + sh(axis, m))
            s.append(acc)
        u = core + dtD * (s[0] * dxi2[0] + s[1] * dxi2[1] + s[2] * dxi2[2])
    return u


def reduce_sum(mf: HostMF, comp: int = 0) -> float:
    off, lo, ext = mf.tables()
    v = np.ascontiguousarray(mf.valid_tab)
    return float(lib().orc_reduce_sum(_p(mf.buf, _f64p), _p(off, _i64p), _p(lo, _i64p), _p(ext, _i64p),
                                      _p(v, _i64p), len(mf.valids), comp))


def reduce_max(mf: HostMF, comp: int = 0) -> float:
    return max(float(np.max(mf.valid_view(u, comp))) for u in range(len(mf.valids)))


def reduce_min(mf: HostMF, comp: int = 0) -> float:
    return min(float(np.min(mf.valid_view(u, comp))) for u in range(len(mf.valids)))


def gsrb_color(phi: HostMF, rhs: HostMF, tiles, color: int, h2: float, nthreads: int = 1) -> None:
    arr = np.ascontiguousarray(tiles if isinstance(tiles, np.ndarray) else tiles_array(tiles))
    po, pl, pe = phi.tables()
    ro, rl, re = rhs.tables()
    lib().orc_gsrb_color(_p(phi.buf, _f64p), _p(po, _i64p), _p(pl, _i64p), _p(pe, _i64p),
                         _p(rhs.buf, _f64p), _p(ro, _i64p), _p(rl, _i64p), _p(re, _i64p),
                         _p(arr, _i64p), len(arr), color, h2, nthreads)


def residual_max(phi: HostMF, rhs: HostMF, tiles, h2: float, nthreads: int = 1) -> float:
    arr = np.ascontiguousarray(tiles if isinstance(tiles, np.ndarray) else tiles_array(tiles))
    po, pl, pe = phi.tables()
    ro, rl, re = rhs.tables()
    return float(lib().orc_residual_max(_p(phi.buf, _f64p), _p(po, _i64p), _p(pl, _i64p), _p(pe, _i64p),
                                        _p(rhs.buf, _f64p), _p(ro, _i64p), _p(rl, _i64p), _p(re, _i64p),
                                        _p(arr, _i64p), len(arr), h2, nthreads))


# --------------------------------------------------------------------------
# Whole-domain periodic restatement (numpy)
# --------------------------------------------------------------------------
def heat_periodic(u: np.ndarray, steps: int, dxi, dtD: float) -> np.ndarray:
    """``u`` (ncomp, nz, ny, nx), fully periodic: ``steps`` forward-Euler
    steps with the flux-form arithmetic of compiled.py:32-81."""
    u = np.array(u, dtype=np.float64, copy=True)
    for _ in range(steps):
        p = np.pad(u, ((0, 0), (1, 1), (1, 1), (1, 1)), mode="wrap")
        c = p[:, 1:-1, 1:-1, 1:-1]
        fxm = (c - p[:, 1:-1, 1:-1, :-2]) * dxi[0]
        fxp = (p[:, 1:-1, 1:-1, 2:] - c) * dxi[0]
        fym = (c - p[:, 1:-1, :-2, 1:-1]) * dxi[1]
        fyp = (p[:, 1:-1, 2:, 1:-1] - c) * dxi[1]
        fzm = (c - p[:, :-2, 1:-1, 1:-1]) * dxi[2]
        fzp = (p[:, 2:, 1:-1, 1:-1] - c) * dxi[2]
        s = (fxp - fxm) * dxi[0] + (fyp - fym) * dxi[1]
        s = s + (fzp - fzm) * dxi[2]
        u = c + dtD * s
    return u


def gsrb_periodic(phi: np.ndarray, rhs: np.ndarray, sweeps: int, h2: float):
    """Whole-domain red-black GS, fully periodic; phi/rhs (nz, ny, nx).
    Returns (phi, max|residual|)."""
    phi = np.array(phi, dtype=np.float64, copy=True)
    n = phi.shape
    k, j, i = np.meshgrid(np.arange(n[0]), np.arange(n[1]), np.arange(n[2]), indexing="ij")
    colour = (i + j + k) & 1

    def nsum(p):
        q = np.pad(p, 1, mode="wrap")
        s = q[1:-1, 1:-1, :-2] + q[1:-1, 1:-1, 2:]
        s = s + q[1:-1, :-2, 1:-1]
        s = s + q[1:-1, 2:, 1:-1]
        s = s + q[:-2, 1:-1, 1:-1]
        s = s + q[2:, 1:-1, 1:-1]
        return s

    for _ in range(sweeps):
        for col in (0, 1):
            upd = (nsum(phi) + h2 * rhs) / 6.0
            phi = np.where(colour == col, upd, phi)
    r = rhs + (nsum(phi) - 6.0 * phi) / h2
    return phi, float(np.max(np.abs(r)))


# --------------------------------------------------------------------------
# Literal restatement of the reference plan builder, O(units^2)
# --------------------------------------------------------------------------
def ref_fill_tags(valids, domain, periodic, nghost):
    """Tags (du, dst lo/hi, su, src lo/hi, shift) exactly as
    level.py:240-287 enumerates them.  ``valids``/``domain``: (lo, hi)."""
    valids = [(tuple(v[0]), tuple(v[1])) for v in valids]
    if nghost == 0:
        return []
    L = [domain[1][d] - domain[0][d] + 1 for d in range(3)]
    per_dim = []
    for d in range(3):
        vals = [0]
        if periodic[d]:
            for k in range(1, ceil(nghost / L[d]) + 1):
                vals += [k * L[d], -k * L[d]]
        per_dim.append(vals)
    shifts = [(a, b, c) for c in per_dim[2] for b in per_dim[1] for a in per_dim[0]]
    shifts.sort(key=lambda s: s != (0, 0, 0))

    def isect(a, b):
        lo = tuple(max(a[0][d], b[0][d]) for d in range(3))
        hi = tuple(min(a[1][d], b[1][d]) for d in range(3))
        return None if any(hi[d] < lo[d] for d in range(3)) else (lo, hi)

    def slabs(v):
        lo = [x - nghost for x in v[0]]
        hi = [x + nghost for x in v[1]]
        out = []
        for d in range(3):
            if lo[d] < v[0][d]:
                h = list(hi)
                h[d] = v[0][d] - 1
                out.append((tuple(lo), tuple(h)))
                lo[d] = v[0][d]
            if hi[d] > v[1][d]:
                l2 = list(lo)
                l2[d] = v[1][d] + 1
                out.append((tuple(l2), tuple(hi)))
                hi[d] = v[1][d]
        return out

    tags = []
    for du, dv in enumerate(valids):
        for g in slabs(dv):
            for s in shifts:
                for su, sv in enumerate(valids):
                    shv = (tuple(sv[0][d] + s[d] for d in range(3)), tuple(sv[1][d] + s[d] for d in range(3)))
                    x = isect(g, shv)
                    if x is None:
                        continue
                    src = (tuple(x[0][d] - s[d] for d in range(3)), tuple(x[1][d] - s[d] for d in range(3)))
                    tags.append((du, x, su, src, s))
    return tags


def expected_ghosts(valids, abox_lo, abox_hi, domain, periodic, field, sentinel):
    """Expected contents of one unit's allocation box after FillBoundary
    when every valid cell holds ``field(i, j, k)`` and every ghost started
    at ``sentinel``: periodic image if some valid box covers it, else the
    sentinel (reference tests/test_acceptance.py:99-121 logic).  Returns an
    (nx, ny, nz) array."""
    axes = [np.arange(abox_lo[d], abox_hi[d] + 1) for d in range(3)]
    W = list(np.meshgrid(*axes, indexing="ij"))
    n = [domain[1][d] - domain[0][d] + 1 for d in range(3)]
    for d in range(3):
        if periodic[d]:
            W[d] = domain[0][d] + (W[d] - domain[0][d]) % n[d]
    covered = np.zeros(W[0].shape, dtype=bool)
    for (lo, hi) in valids:
        m = np.ones(W[0].shape, dtype=bool)
        for d in range(3):
            m &= (W[d] >= lo[d]) & (W[d] <= hi[d])
        covered |= m
    return np.where(covered, field(W[0], W[1], W[2]), sentinel)
