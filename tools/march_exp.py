"""Time the fused heat step (the bench kernel) for column heights / CTA counts,
as the runner drives it: graph-captured pairs a->b (forward), b->a (reverse).

    python tools/march_exp.py [--config C2] [--shapes 16:296,16:444] [--reps 50]

Set TILEMESH_LIB to time another build of the library (experiment variants
are compiled outside the package and loaded this way).  Prints one line per
shape: microseconds per step and the algorithmic GB/s (16 B per cell).
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.march import FusedHalo  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    cfg = arg("--config", "C2")
    reps = int(arg("--reps", "50"))
    shapes = [tuple(None if v == "-" else int(v) for v in s.split(":")) for s in arg("--shapes", "-:-").split(",")]
    w = tm.CONFIGS[cfg]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    a = tm.MultiFab(ba, w.ncomp, w.nghost)
    a.from_global(torch.rand((w.ncomp,) + (w.n,) * 3, dtype=torch.float64, device="cuda"))
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    cells = w.cells * w.ncomp
    lib = os.environ.get("TILEMESH_LIB", "package")
    for rows, nctas in shapes:
        fh = FusedHalo(a, b, geom, rows, nctas)
        fh.prime(a)

        def pair():
            fh.step(b, a, p, reverse=False)
            fh.step(a, b, p, reverse=True)

        pair()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                pair()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(400_000)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (4 * reps * 2)
        print(f"{lib} {cfg} rows={rows} nctas={fh.plan.nctas} cols={fh.plan.ncolumns}: {us:.2f} us/step "
              f"{16 * cells / us / 1e3:.0f} GB/s alg", flush=True)
        del g


if __name__ == "__main__":
    main()
