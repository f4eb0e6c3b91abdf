"""The device checksum (``tm_reduce_sum``) against the reference's serial sum
on adversarial data.  The kernel evaluates the per-grid chain T <- fl(T + v)
warp-parallel in integer arithmetic wherever the roundings provably match and
serially elsewhere, so every case here must be bit-identical to the oracle's
strictly serial C loop (level.py:183-190, compiled.py:20-29): binade changes,
sign changes and cancellation, exact ties, subnormals, +-0, huge magnitudes
outside the fast path's exponent window, Inf and NaN; rows that the kernel
streams by bulk copies (x extents a multiple of 8) and by loads (other
extents, or rows longer than a ring stage)."""

import struct

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def fields(n, rng):
    k = int(np.prod(n))
    out = {
        "u01": rng.random(k),
        "signed": rng.standard_normal(k),
        "mixed_magnitudes": rng.standard_normal(k) * 10.0 ** rng.integers(-30, 30, k),
        "eighths_ties": rng.integers(0, 8, k) * 0.25 + 0.125,
        "half_integers": rng.integers(-50, 50, k) * 0.5,
        "powers_of_two": 2.0 ** rng.integers(-60, 60, k),
        "cancellation": np.where(rng.random(k) < 0.5, 1e16, -1e16) * rng.random(k) + rng.random(k),
        "subnormal": rng.random(k) * 1e-310,
        "huge": rng.random(k) * 1e300,
        "zeros": np.zeros(k),
        "neg_zeros": np.full(k, -0.0),
        "large_then_small": np.concatenate([[2.0 ** 53], rng.random(k - 1)]),
        "ramp_crossing_zero": np.linspace(-3.0, 3.0, k) + rng.random(k) * 1e-3,
    }
    inf = rng.random(k)
    inf[k // 3] = np.inf
    out["inf"] = inf
    nan = rng.random(k)
    nan[k // 2] = np.nan
    out["nan"] = nan
    return {name: v.reshape((1,) + tuple(reversed(n))) for name, v in out.items()}


def same(a, b):
    return struct.pack("<d", a) == struct.pack("<d", b) or (np.isnan(a) and np.isnan(b))


@pytest.mark.parametrize("domain,chop", [
    ((48, 24, 16), (24, 12, 8)),   # x extent a multiple of 8: multi-row bulk copies
    ((32, 50, 3), (32, 50, 3)),    # ... with a partial stage at the end of every plane
    ((40, 24, 16), (20, 12, 8)),   # x extent not a multiple of 8: load gather
    ((33, 10, 6), (11, 10, 6)),    # odd x extent
    ((1030, 4, 2), (1030, 4, 2)),  # long odd rows
    ((2056, 3, 2), (2056, 3, 2)),  # rows longer than a ring stage
])
def test_device_checksum_matches_serial_sum(tm, domain, chop):
    rng = np.random.default_rng(7)
    dom = tm.Box((0, 0, 0), tuple(d - 1 for d in domain))
    ba = tm.BoxArray.chop(dom, chop)
    mf = tm.MultiFab(ba, 1, 1)
    h = orc.HostMF(list(ba), 1, 1)
    bad = []
    for name, glob in fields(domain, rng).items():
        mf.from_global(glob)
        h.from_global(glob)
        got, want = mf.reduce_sum(0), orc.reduce_sum(h, 0)
        if not same(got, want):
            bad.append((name, got, want))
    assert not bad, bad


def test_device_checksum_c2_size(tm):
    """One 64^3 grid of the headline shape, values of the heat run's kind."""
    rng = np.random.default_rng(11)
    dom = tm.Box((0, 0, 0), (63, 63, 63))
    ba = tm.BoxArray([dom])
    mf = tm.MultiFab(ba, 1, 1)
    h = orc.HostMF(list(ba), 1, 1)
    for glob in (rng.random((1, 64, 64, 64)), rng.standard_normal((1, 64, 64, 64)) * 1e3):
        mf.from_global(glob)
        h.from_global(glob)
        assert same(mf.reduce_sum(0), orc.reduce_sum(h, 0))
