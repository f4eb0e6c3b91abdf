"""Run a few fused GSRB sweeps of config C4 (for ncu captures).
python tools/gsrb_steps.py [sweeps]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402


def main():
    sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    w = tm.CONFIGS["C4"]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    phi = tm.MultiFab(ba, 1, 1)
    rhs = tm.MultiFab(ba, 1, 0)
    rhs.from_global(tm.make_init(w))
    tm.gsrb_solve(phi, rhs, geom, sweeps, fused=True)
    torch.cuda.synchronize()
    print("residual", tm.residual_maxnorm(phi, rhs, geom))


if __name__ == "__main__":
    main()
