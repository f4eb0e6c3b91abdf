"""wide4 throughput on a C2-shaped problem (256^3, 64^3 boxes, nghost 4):
Kernel W alone, FillBoundary (4 ghost layers) alone, and the reference step
(FB + wide4), and the fused step (Wide4Runner: one launch, face ghosts written
by the epilogue).  python tools/wide4_perf.py [n mgs] [--rows R --nctas N]"""

import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.wide4 import _launch  # noqa: E402
from tools.sweep_shapes import graph_time  # noqa: E402


def arg(name, default=None):
    return int(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def main():
    pos = [a for a in sys.argv[1:] if a.isdigit()]
    n, mgs = (int(pos[0]), int(pos[1])) if len(pos) >= 2 else (256, 64)
    w = dataclasses.replace(tm.CONFIGS["C2"].scaled(n, mgs, 10), nghost=4)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    a = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), 1, 4)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    plan = tm.build_fill_plan(a, geom)
    dt = tm.wide4_stable_dt(1.0, geom.dx)
    co = tm.derive_coeffs8()
    rows, nctas = arg("--rows"), arg("--nctas")
    tm.fill_boundary(a, geom, plan)
    kern = graph_time(lambda: _launch(b, a, geom, 1.0, dt, co, rows, nctas), 10)
    fb = graph_time(lambda: tm.fill_boundary(a, geom, plan), 10)
    step = graph_time(lambda: (tm.fill_boundary(a, geom, plan), _launch(b, a, geom, 1.0, dt, co, rows, nctas),
                               tm.fill_boundary(b, geom, plan), _launch(a, b, geom, 1.0, dt, co, rows, nctas)), 5) / 2
    r = tm.Wide4Runner(a, geom, 1.0, dt, co, fused=True)
    r.advance(2)
    fused = graph_time(lambda: (r._step(r.a, r.b), r._step(r.b, r.a)), 5) / 2
    r.close()
    cells = w.cells
    ghosts = sum(t.dst_box.ncells for t in plan.tags)
    print(f"wide4 {n}^3 mgs {mgs}: kernel {kern * 1e3:.1f} us ({cells / kern / 1e6:.1f} G cell/s, "
          f"{16 * cells / kern / 1e6:.0f} GB/s alg) | FB {fb * 1e3:.1f} us ({ghosts} ghost cells, "
          f"{16 * ghosts / fb / 1e6:.0f} GB/s) | step {step * 1e3:.1f} us ({cells / step / 1e6:.1f} G cell/s) | "
          f"fused step {fused * 1e3:.1f} us ({cells / fused / 1e6:.1f} G cell/s)")


if __name__ == "__main__":
    main()
