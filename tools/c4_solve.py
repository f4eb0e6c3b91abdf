"""C4 GSRB solve timing (50 sweeps incl. split/merge and closing fill), CUDA events:
python tools/c4_solve.py"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402


def main():
    w = tm.CONFIGS["C4"]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    phi = tm.MultiFab(ba, 1, 1)
    rhs = tm.MultiFab(ba, 1, 0)
    rhs.from_global(tm.make_init(w))
    tm.gsrb_solve(phi, rhs, geom, 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tm.gsrb_solve(phi, rhs, geom, w.steps)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / w.steps * 1e3
    print(f"C4 solve {w.steps} sweeps: {us:.1f} us/sweep, {w.cells / us / 1e3:.1f} G cell-upd/s, "
          f"frac {24 * w.cells / (us * 1e-6) / 1e9 / 6553.6:.3f} (24 B basis)")


if __name__ == "__main__":
    main()
