"""Time the phases of bench.py's end-to-end job (config C2) separately.
python tools/e2e_phases.py"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.runner import HeatRunner  # noqa: E402


def main():
    w = tm.CONFIGS["C2"]
    dev = torch.device("cuda", 0)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    glob = torch.from_numpy(tm.make_init(w)).pin_memory()
    host_out = torch.empty_like(glob).pin_memory()
    mf = tm.MultiFab(ba, w.ncomp, w.nghost)
    mf.from_global(glob.to(dev))
    r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx))
    r.advance(4)
    state = {}
    phases = {
        "h2d": lambda: state.__setitem__("g", glob.to(dev, non_blocking=True)),
        "from_global": lambda: r.a.from_global(state["g"]),
        "advance100": lambda: (r.reset(), state.__setitem__("out", r.advance(w.steps))),
        "reduce": lambda: state.__setitem__("cs", state["out"].reduce_sum_device()),
        "to_global": lambda: state.__setitem__("tg", state["out"].to_global()),
        "d2h": lambda: host_out.copy_(state["tg"]),
        "csum_item": lambda: float(state["cs"].item()),
    }
    side = torch.cuda.Stream(dev)

    def overlapped():
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            state["cs"] = state["out"].reduce_sum_device()
        host_out.copy_(state["out"].to_global())
        torch.cuda.current_stream().wait_stream(side)
        float(state["cs"].item())
    phases["reduce||to_global+d2h"] = overlapped
    for rep in range(3):
        line = []
        for name, fn in phases.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            line.append(f"{name} {e0.elapsed_time(e1):.3f}")
        print(" | ".join(line))


if __name__ == "__main__":
    main()
