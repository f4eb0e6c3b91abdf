"""Two-steps-per-launch kernel (tm_heat_march2) on a config with nghost 2:
kernel alone, FillBoundary (2 layers) alone, and FB + kernel per 2 steps.
python tools/march2_perf.py [--config C2] [--nctas N]"""

import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.march import FusedHalo2, heat_march2  # noqa: E402
from tools.sweep_shapes import graph_time  # noqa: E402


def main():
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "C2"
    nctas = int(sys.argv[sys.argv.index("--nctas") + 1]) if "--nctas" in sys.argv else None
    rows = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else None
    w = dataclasses.replace(tm.CONFIGS[cfg], nghost=max(2, tm.CONFIGS[cfg].nghost))
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    a = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), w.ncomp, w.nghost)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    plan = tm.build_fill_plan(a, geom)
    tm.fill_boundary(a, geom, plan)
    cells = w.cells * w.ncomp
    kern = graph_time(lambda: heat_march2(b, a, p, max_rows=rows, nctas=nctas), 10)
    fb = graph_time(lambda: tm.fill_boundary(a, geom, plan), 10)
    pair = graph_time(lambda: (tm.fill_boundary(a, geom, plan), heat_march2(b, a, p, max_rows=rows, nctas=nctas),
                               tm.fill_boundary(b, geom, plan), heat_march2(a, b, p, max_rows=rows, nctas=nctas)), 5) / 2
    fh = FusedHalo2(a, b, geom, nctas, rows, packed="--packed" in sys.argv)
    fh.prime(a, plan)
    fused = graph_time(lambda: (fh.step2(b, a, p), fh.step2(a, b, p)), 5) / 2
    print(f"{cfg} fused two-step launch (scatter) {fused * 1e3:.1f} us = {fused * 1e3 / 2:.1f} us/step, "
          f"{2 * cells / fused / 1e6:.1f} G cell-upd/s")
    print(f"{cfg} two-step kernel {kern * 1e3:.1f} us ({2 * cells / kern / 1e6:.1f} G cell-upd/s, "
          f"{16 * cells / kern / 1e6:.0f} GB/s per launch) | FB(ng {w.nghost}) {fb * 1e3:.1f} us | "
          f"FB + kernel {pair * 1e3:.1f} us per 2 steps = {2 * cells / pair / 1e6:.1f} G cell-upd/s")


if __name__ == "__main__":
    main()
