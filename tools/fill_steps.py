"""FillBoundary loop on a config (for ncu): python tools/fill_steps.py [C2] [reps]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    w = tm.CONFIGS[cfg]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    mf = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), w.ncomp, w.nghost)
    mf.from_global(tm.make_init(w))
    plan = tm.build_fill_plan(mf, geom)
    if "--time" in sys.argv:
        from tools.sweep_shapes import graph_time

        ms = graph_time(lambda: tm.fill_boundary(mf, geom, plan), 20)
        ghosts = sum(t.dst_box.ncells for t in plan.tags) * w.ncomp
        print(f"{cfg} FillBoundary {ms * 1e3:.1f} us, {ghosts} ghost cells, {16 * ghosts / ms / 1e6:.0f} GB/s")
        return
    for _ in range(reps):
        tm.fill_boundary(mf, geom, plan)
    torch.cuda.synchronize()
    print("done", cfg, reps)


if __name__ == "__main__":
    main()
