"""Time the pieces of the reference-shaped loop (fill_boundary; heat_step) on C2
as graph replays: the fast fill (edge/corner copies; the faces are written by
the next heat_step's sweep), the face copies a settle would cost, and the whole
loop.  python tools/refloop_perf.py [--config C2]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.multifab import _xh_fill  # noqa: E402
from paper_1604_03570_b200.runner import HeatRunner  # noqa: E402
from tools.sweep_shapes import graph_time  # noqa: E402


def main():
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "C2"
    w = tm.CONFIGS[cfg]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    a = tm.MultiFab(ba, w.ncomp, w.nghost)
    a.from_global(torch.rand((w.ncomp,) + (w.n,) * 3, dtype=torch.float64, device="cuda"))
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    plan = tm.build_fill_plan(a, geom)
    cells = w.cells * w.ncomp
    for _ in range(3):  # reach the fast path on both fields
        tm.fill_boundary(a, geom, plan)
        tm.heat_step(b, a, geom, p)
        tm.fill_boundary(b, geom, plan)
        tm.heat_step(a, b, geom, p)
    assert a.xh_current()
    edges, faces, _, _ = _xh_fill(a, plan, geom)

    def edge_part():
        edges.run(a.gptr, a.layout.side(), a.ptr, a.layout.side(), a.stream())

    def face_part():  # what settling deferred faces costs (not on the loop's path)
        faces.run(a.gptr, a.layout.side(), a.ptr, a.layout.side(), a.stream())

    def pair():
        tm.fill_boundary(a, geom, plan)
        tm.heat_step(b, a, geom, p)
        tm.fill_boundary(b, geom, plan)
        tm.heat_step(a, b, geom, p)

    res = {"edge/corner copies (the fill on the loop's path)": graph_time(edge_part, 20),
           "y/z face copies (settling deferred faces)": graph_time(face_part, 20)}
    a._xh_key = a.valid_key()  # the timing loops above do not change valid cells
    # the loop as a drop-in caller issues it (eager Python), and as HeatRunner(fused=False)
    # replays it (4-step graphs: the packed-halo buffers repeat every two steps per field)
    for _ in range(2):
        pair()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        pair()
    e1.record()
    torch.cuda.synchronize()
    res["loop step, eager Python"] = e0.elapsed_time(e1) / 40
    r = HeatRunner(a, geom, p, None, plan, fused=False)
    r.advance(8)
    torch.cuda.synchronize()
    e0.record()
    r.advance(40, finalize=False)
    e1.record()
    torch.cuda.synchronize()
    res["loop step (fill + heat_step)"] = e0.elapsed_time(e1) / 40
    for k, ms in res.items():
        print(f"{cfg} {k}: {ms * 1e3:.1f} us")
    step = res["loop step (fill + heat_step)"]
    print(f"{cfg} reference loop (HeatRunner graph): {cells / step / 1e6:.1f} G cell-upd/s, "
          f"{16 * cells / step / 1e6 / 6553.6:.3f} of 6553.6 GB/s")


if __name__ == "__main__":
    main()
