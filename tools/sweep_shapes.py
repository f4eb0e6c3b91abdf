"""Time the heat sweep and the FillBoundary kernel alone for several CTA
block shapes (CUDA graph of N launches, CUDA events), C2 by default.

    python tools/sweep_shapes.py [--config C2] [--reps 20]
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402


def graph_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (3 * reps)


def main():
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "C2"
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 20
    w = tm.CONFIGS[cfg]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    a = tm.MultiFab(ba, w.ncomp, w.nghost)
    a.from_global(tm.make_init(w))
    b = a.clone_empty()
    plan = tm.build_fill_plan(a, geom)
    p = tm.HeatParams.stable(1.0, geom.dx)
    cells = w.cells * w.ncomp
    ms = graph_time(lambda: tm.fill_boundary(a, geom, plan), reps)
    ghost = sum(t.dst_box.ncells for t in plan.tags) * w.ncomp
    print(f"{cfg} fill: {ms * 1e3:.1f} us  ({16 * ghost / ms / 1e6:.0f} GB/s of ghost r+w)")
    shapes = [w.tile_size, (1024, 8, 1024), (1024, 16, 1024), (1024, 32, 1024), (1024, 16, 32), (1024, 16, 16),
              (1024, 4, 1024), (1024, 64, 1024)]
    for ts in shapes:
        for zm in (False,):
            sched = tm.build_schedule(a, ts)
            try:
                ms = graph_time(lambda: tm.heat_step(b, a, geom, p, sched, zmerge=zm), reps)
            except ValueError as e:
                print(ts, "skip", e)
                continue
            nb = tm.multifab.schedule_sweep_plan(a, sched, zm).nblocks
            print(f"{cfg} sweep tile {ts} zmerge={zm} ctas={nb}: {ms * 1e3:.1f} us "
                  f"{16 * cells / ms / 1e6:.0f} GB/s alg ({cells / ms / 1e6:.1f} G cell/s)")


if __name__ == "__main__":
    main()
