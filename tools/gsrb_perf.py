"""Per-pass timing of the GSRB kernels on config C4 (256^3, 64^3 boxes):
in-place fused (tm_gsrb_march) vs colour-split (tm_gsrb_split_pass).
python tools/gsrb_perf.py [--rows R] [--nctas N]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.march import FusedGSRB, SplitGSRB  # noqa: E402
from tools.sweep_shapes import graph_time  # noqa: E402


def arg(name):
    return int(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else None


def main():
    w = tm.CONFIGS["C4"]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    phi = tm.MultiFab(ba, 1, 1)
    rhs = tm.MultiFab(ba, 1, 0)
    rhs.from_global(tm.make_init(w))
    cells = w.cells
    fg = FusedGSRB(phi, rhs, geom, arg("--rows"), arg("--nctas"))
    fg.prime()
    t_in = graph_time(fg.sweep, 10) / 2
    sg = SplitGSRB(phi, rhs, geom, arg("--rows"), arg("--nctas"))
    sg.prime()
    t_sp = graph_time(sg.sweep, 10) / 2
    t_prime = graph_time(sg.prime, 3)
    t_fin = graph_time(sg.finalize, 3)
    print(f"C4 in-place fused pass {t_in * 1e3:.1f} us ({24 * cells / t_in / 1e6:.0f} GB/s on 24 B/cell) | "
          f"colour-split pass {t_sp * 1e3:.1f} us ({12 * cells / t_sp / 1e6:.0f} GB/s moved) | "
          f"split prime {t_prime * 1e3:.0f} us, merge+fill {t_fin * 1e3:.0f} us")


if __name__ == "__main__":
    main()
