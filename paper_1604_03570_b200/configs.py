"""BASELINE.json workloads C1-C5 and their seeded synthetic inputs.

BASELINE.json names no public dataset: its five configs are the inputs
(SURVEY.md §8d).  Conventions shared by every config:

* domain ``[0, n-1]^3``, fully periodic, ``dx = 1/n``, ``D = 1``,
  ``dt = HeatParams.stable(1.0, dx).dt``;
* boxes from ``BoxArray.chop(domain, max_grid_size)``;
* random draws from ``np.random.default_rng(seed)`` in global x-fastest
  order, component by component, generated once on the host in float64;
  the CPU oracle and the device consume the same host array;
* cell centres ``x = (i + 0.5) * dx``.

Global arrays have shape ``(ncomp, nz, ny, nx)`` (C order, x fastest).

``det_exp`` evaluates ``exp`` with IEEE basic operations only (Cody-Waite
reduction + Taylor polynomial + ldexp, <= 2 ulp), so the Gaussian inits are
bit-identical on every host; numpy's own ``exp`` dispatches to
host-specific SIMD code (AVX512F here) whose last-bit results differ from
other hosts, which would make golden hashes host-dependent.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .box import Box


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    max_grid_size: int
    nghost: int
    ncomp: int
    tile_size: tuple
    steps: int
    kernel: str  # "heat" or "gsrb"
    init: str
    seed: int = 0
    nz: int | None = None  # z extent when the domain is not a cube (weak-scaled slabs)

    @property
    def domain(self) -> Box:
        return Box((0, 0, 0), (self.n - 1, self.n - 1, (self.nz or self.n) - 1))

    @property
    def dx(self) -> float:
        return 1.0 / self.n

    @property
    def cells(self) -> int:
        return self.n * self.n * (self.nz or self.n)

    def weak(self, ranks: int) -> "Workload":
        """Weak-scaled slab domain: n x n x (L * max_grid_size * ranks), L box
        layers per rank -- the config's per-GPU share at 8 GPUs (C5: 4 layers
        of 32^3 boxes, so 8 ranks hold the full C5; C2 / C3: one layer).
        Uniform random init (the values do not change any code path)."""
        layers = max(1, self.n // self.max_grid_size // 8)
        return Workload(f"{self.name}-weak{ranks}", self.n, self.max_grid_size, self.nghost, self.ncomp,
                        self.tile_size, self.steps, self.kernel, "uniform", self.seed,
                        nz=layers * self.max_grid_size * ranks)

    def scaled(self, n: int, max_grid_size: int | None = None, steps: int | None = None) -> "Workload":
        """Same workload shape at a smaller domain (parity tests)."""
        return Workload(self.name + f"@{n}", n, max_grid_size or self.max_grid_size, self.nghost,
                        self.ncomp, self.tile_size, steps if steps is not None else self.steps,
                        self.kernel, self.init, self.seed)


CONFIGS = {
    "C1": Workload("C1", 64, 32, 1, 1, (1024, 8, 8), 10, "heat", "gauss_noise"),
    "C2": Workload("C2", 256, 64, 1, 1, (1024, 8, 8), 100, "heat", "gauss_noise"),
    "C3": Workload("C3", 512, 128, 2, 4, (1024, 16, 16), 50, "heat", "uniform_bump"),
    "C4": Workload("C4", 256, 64, 1, 1, (1024, 8, 8), 50, "gsrb", "poisson_rhs"),
    "C5": Workload("C5", 1024, 32, 2, 2, (1024, 8, 8), 20, "heat", "uniform"),
}

# Gaussian-bump centres for the C3 components (builder's choice, documented
# in DESIGN.md): octant centres on a diagonal-ish pattern.
C3_CENTRES = [(0.25, 0.25, 0.25), (0.75, 0.25, 0.25), (0.25, 0.75, 0.75), (0.75, 0.75, 0.5)]

_LN2_HI = 6.93147180369123816490e-01  # 0x3FE62E42FEE00000: exact n*LN2_HI for |n| < 2^11
_LN2_LO = 1.90821492927058770002e-10
_INV_LN2 = 1.44269504088896338700e00


def det_exp(x: np.ndarray) -> np.ndarray:
    """Host-independent exp for float64 arrays with ``-700 < x < 700``."""
    x = np.asarray(x, dtype=np.float64)
    n = np.rint(x * _INV_LN2)
    r = (x - n * _LN2_HI) - n * _LN2_LO
    # Taylor series to degree 13 on |r| <= 0.347: truncation < 1e-19 relative
    p = np.full_like(r, 1.0 / math.factorial(13))
    for k in range(12, -1, -1):
        p = p * r
        p = p + 1.0 / math.factorial(k)
    return np.ldexp(p, n.astype(np.int64))


def _centres(n: int):
    c = (np.arange(n, dtype=np.float64) + 0.5) * (1.0 / n)
    return c


def gaussian(n: int, centre=(0.5, 0.5, 0.5), width: float = 0.01) -> np.ndarray:
    """``exp(-((x-cx)^2+(y-cy)^2+(z-cz)^2)/width)`` on the cell centres, (nz, ny, nx)."""
    c = _centres(n)
    dx2 = (c - centre[0]) ** 2
    dy2 = (c - centre[1]) ** 2
    dz2 = (c - centre[2]) ** 2
    r2 = (dx2[None, None, :] + dy2[None, :, None]) + dz2[:, None, None]
    return det_exp(-(r2 / width))


def make_init(w: Workload) -> np.ndarray:
    """Global initial data ``(ncomp, nz, ny, nx)`` for a workload (phi, or
    rhs for the Poisson config)."""
    n = w.n
    if w.nz not in (None, n) and w.init != "uniform":
        raise ValueError(f"init {w.init!r} is defined on cubic domains only")
    rng = np.random.default_rng(w.seed)
    shape = (n, n, n)
    if w.init == "gauss_noise":
        # phi = 1 + exp(-r^2/0.01) + 1e-3 * U(-1, 1)
        noise = rng.uniform(-1.0, 1.0, size=n ** 3).reshape(shape)
        phi = (1.0 + gaussian(n)) + 1e-3 * noise
        return phi.reshape((1,) + shape)
    if w.init == "uniform":
        shape = ((w.nz or n), n, n)
        out = np.empty((w.ncomp,) + shape)
        for c in range(w.ncomp):
            out[c] = rng.random(int(np.prod(shape))).reshape(shape)
        return out
    if w.init == "uniform_bump":
        out = np.empty((w.ncomp,) + shape)
        for c in range(w.ncomp):
            out[c] = rng.random(n ** 3).reshape(shape) + gaussian(n, C3_CENTRES[c % 4])
        return out
    if w.init == "poisson_rhs":
        rhs = rng.uniform(-1.0, 1.0, size=n ** 3)
        mean = math.fsum(rhs) / rhs.size  # exactly rounded sum: host-independent
        return (rhs - mean).reshape((1,) + shape)
    if w.init == "cosine":
        c = _centres(n)
        f = np.cos(2.0 * np.pi * c)
        return (f[None, None, :] * f[None, :, None] * f[:, None, None]).reshape((1,) + shape)
    raise ValueError(f"unknown init {w.init!r}")
