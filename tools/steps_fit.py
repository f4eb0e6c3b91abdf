"""Fixed vs per-step cost of the bench's timed region: K fused C2 steps between CUDA events
for several K and several lengths of the device sleep queued before the first event.

    python tools/steps_fit.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.runner import HeatRunner  # noqa: E402


def main():
    w = tm.CONFIGS["C2"]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    mf = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), w.ncomp, w.nghost)
    mf.from_global(torch.rand((w.ncomp,) + (w.n,) * 3, dtype=torch.float64, device="cuda"))
    r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx))
    r.advance(2000, finalize=False)
    stream = torch.cuda.current_stream()
    for sleep in (400_000, 4_000_000):
        for k in (20, 40, 100, 400, 2000):
            r.advance(k, finalize=False)
            ts = []
            for _ in range(7):
                r.advance(400, finalize=False)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(sleep)
                e0.record(stream)
                r.advance(k, finalize=False)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            print(f"sleep {sleep:>8} K {k:>5}: min {ts[0] / k:.2f} med {ts[3] / k:.2f} max {ts[-1] / k:.2f} us/step;"
                  f" total med {ts[3]:.0f} us", flush=True)


if __name__ == "__main__":
    main()
