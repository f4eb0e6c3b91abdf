"""Time the column-march sweep (STD halos) and the fused step for several
column heights / CTA counts.  python tools/march_perf.py [--config C2]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200 import march  # noqa: E402
from tools.sweep_shapes import graph_time  # noqa: E402


def main():
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "C2"
    w = tm.CONFIGS[cfg]
    if "--scaled" in sys.argv:
        k = sys.argv.index("--scaled")
        w = w.scaled(int(sys.argv[k + 1]), int(sys.argv[k + 2]))
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    a = tm.MultiFab(ba, w.ncomp, w.nghost)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    cells = w.cells * w.ncomp
    nsm = march.sm_count(a.device)
    for rows in (() if "--fused-only" in sys.argv else (None, 32, 16)):
        for mult in (None, 1, 2, 3):
            nctas = None if mult is None else nsm * mult
            try:
                ms = graph_time(lambda: march.heat_march(b, a, p, max_rows=rows, nctas=nctas), 20)
            except Exception as e:  # noqa: BLE001
                print(f"{cfg} march rows={rows} nctas={nctas}: {e}")
                continue
            pl = march.march_plan(a, False, rows, nctas)
            print(f"{cfg} march-std rows={rows} nctas={pl.nctas} cols={pl.ncolumns}: {ms * 1e3:.1f} us "
                  f"{16 * cells / ms / 1e6:.0f} GB/s alg ({cells / ms / 1e6:.1f} G cell/s)")
    for rows in (None, 32, 16, 14, 12, 8):
        for mult in ((None,) if "--fused-only" in sys.argv else (None, 2, 3, 4)):
            nctas = None if mult is None else nsm * mult
            try:
                fh = march.FusedHalo(a, b, geom, rows, nctas)
                fh.prime(a)
                ms = graph_time(lambda: (fh.step(b, a, p), fh.step(a, b, p)), 10) / 2
                msr = graph_time(lambda: (fh.step(b, a, p), fh.step(a, b, p, reverse=True)), 10) / 2
            except Exception as e:  # noqa: BLE001
                print(f"{cfg} fused rows={rows} nctas={nctas}: {e}")
                continue
            print(f"{cfg} fused-step rows={rows} nctas={fh.plan.nctas}: {ms * 1e3:.1f} us "
                  f"{16 * cells / ms / 1e6:.0f} GB/s alg ({cells / ms / 1e6:.1f} G cell/s); "
                  f"alternating direction {msr * 1e3:.1f} us ({cells / msr / 1e6:.1f} G cell/s)")


if __name__ == "__main__":
    main()


def packed_noscatter(cfg="C2", rows=16, nctas=296):
    """PACKED x halos, no scatter (isolates the epilogue's cost)."""
    from paper_1604_03570_b200 import _native

    w = tm.CONFIGS[cfg]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    a = tm.MultiFab(ba, w.ncomp, w.nghost)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    fh = march.FusedHalo(a, b, geom, rows, nctas)
    fh.prime(a)
    c = p.coefficients()

    def go():
        _native.check(_native.load().tm_heat_march(fh.plan.handle, a.layout.to_c(), a.ptr, b.ptr, a.ncomp, c[0], c[1],
                                                   c[2], c[3], _native.HALO_PACKED, fh.xh[id(a)].data_ptr(), None, None, 0,
                                                   a.stream()), "m")
    ms = graph_time(go, 20)
    print(f"{cfg} packed-noscatter rows={rows} nctas={nctas}: {ms * 1e3:.1f} us")


if "--noscatter" in sys.argv:
    for r, n in ((16, 296), (16, 592), (8, 444)):
        packed_noscatter("C2", r, n)
