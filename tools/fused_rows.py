"""C2 fused step (graph-replayed alternating pairs) for a given column height / CTA count:
python tools/fused_rows.py ROWS NCTAS"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200 import march  # noqa: E402
from tools.sweep_shapes import graph_time  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "None" else None
    nctas = int(sys.argv[2]) if len(sys.argv) > 2 else None
    w = tm.CONFIGS[os.environ.get("CFG", "C2")]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    a = tm.MultiFab(ba, w.ncomp, w.nghost)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    fh = march.FusedHalo(a, b, geom, rows, nctas)
    fh.prime(a)
    ms = graph_time(lambda: (fh.step(b, a, p), fh.step(a, b, p, reverse=True)), 20) / 2
    cells = w.cells * w.ncomp
    print(f"{w.name} fused rows={rows} nctas={fh.plan.nctas}: {ms * 1e3:.1f} us/step "
          f"(frac {16 * cells / ms / 1e6 / 6553.6:.3f})")


if __name__ == "__main__":
    main()
