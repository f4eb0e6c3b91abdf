"""Time the device checksum (tm_reduce_sum) on C2-shaped grids for a few
value distributions.  python tools/reduce_perf.py"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402


def main():
    w = tm.CONFIGS["C2"]
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    mf = tm.MultiFab(ba, 1, 1)
    rng = np.random.default_rng(0)
    shape = (1, w.n, w.n, w.n)
    cases = {"init (gauss+noise)": tm.make_init(w), "u01": rng.random(shape), "zeros": np.zeros(shape),
             "signed normal": rng.standard_normal(shape)}
    for name, g in cases.items():
        mf.from_global(g)
        for _ in range(2):
            mf.reduce_sum_device()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            mf.reduce_sum_device()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:20s} {e0.elapsed_time(e1) / 5:.3f} ms  ({len(ba)} grids of {ba[0].ncells} cells)")


if __name__ == "__main__":
    main()
