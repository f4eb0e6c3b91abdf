"""Eager loop for ncu: python tools/march_steps.py [std|fused] [steps] [--rows R] [--nctas N] [--config C2]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200 import march  # noqa: E402


def arg(name, default=None, conv=int):
    return conv(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 6
    rows, nctas = arg("--rows"), arg("--nctas")
    w = tm.CONFIGS[arg("--config", "C2", str)]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    a = tm.MultiFab(ba, w.ncomp, w.nghost)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    plan = tm.build_fill_plan(a, geom)
    if mode == "fused":
        fh = march.FusedHalo(a, b, geom, rows, nctas)
        fh.prime(a, plan)
        for _ in range(steps):
            fh.step(b, a, p)
            a, b = b, a
    else:
        for _ in range(steps):
            tm.fill_boundary(a, geom, plan)
            march.heat_march(b, a, p, max_rows=rows, nctas=nctas)
            a, b = b, a
    torch.cuda.synchronize()
    print("done", mode, steps)


if __name__ == "__main__":
    main()
