"""Timeline of bench.py's pipelined e2e (two C2 jobs in flight on two
streams): per-job event times (ms from the start) of upload / steps /
gather / download / checksum.  python tools/e2e_pipeline.py [--jobs 8]"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.runner import HeatRunner  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=8)
    ap.add_argument("--skip", default="", help="comma list of phases to leave out: h2d,csum,d2h,gather")
    args = ap.parse_args()
    skip = set(args.skip.split(","))
    w = tm.CONFIGS["C2"]
    dev = torch.device("cuda", 0)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    glob = torch.from_numpy(tm.make_init(w)).pin_memory()
    p = tm.HeatParams.stable(1.0, geom.dx)
    runners = []
    for _ in range(2):
        mf = tm.MultiFab(ba, w.ncomp, w.nghost)
        mf.from_global(glob.to(dev))
        runners.append(HeatRunner(mf, geom, p))
    streams = [torch.cuda.Stream(dev) for _ in range(2)]
    sides = [torch.cuda.Stream(dev) for _ in range(2)]
    dev_in = [torch.empty_like(glob, device=dev) for _ in range(2)]
    dev_out = [torch.zeros_like(glob, device=dev) for _ in range(2)]
    host = [torch.empty_like(glob).pin_memory() for _ in range(2)]
    marks = []

    def ev(st):
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    import time
    host_t = []

    def job(j):
        r, st, sd = runners[j % 2], streams[j % 2], sides[j % 2]
        m = {}
        ht = [time.perf_counter()]
        with torch.cuda.stream(st):
            st.wait_stream(sd)
            m["start"] = ev(st)
            if "h2d" not in skip:
                dev_in[j % 2].copy_(glob, non_blocking=True)
            m["h2d"] = ev(st)
            ht.append(time.perf_counter())
            r.a.from_global(dev_in[j % 2])
            ht.append(time.perf_counter())
            r.reset()
            o = r.advance(w.steps)
            ht.append(time.perf_counter())
            m["steps"] = ev(st)
            if "gather" not in skip:
                o.to_global(out=dev_out[j % 2])
            ht.append(time.perf_counter())
            m["gather"] = ev(st)
            sd.wait_stream(st)
            with torch.cuda.stream(sd):
                if "csum" not in skip:
                    o.reduce_sum_device()
                m["csum"] = ev(sd)
            ht.append(time.perf_counter())
            if "d2h" not in skip:
                host[j % 2].copy_(dev_out[j % 2], non_blocking=True)
            m["d2h"] = ev(st)
            ht.append(time.perf_counter())
        marks.append(m)
        host_t.append([1e3 * (b - a) for a, b in zip(ht, ht[1:])])

    for j in range(2):
        job(j)
    torch.cuda.synchronize()
    marks.clear()
    t0 = ev(torch.cuda.current_stream())
    for s in streams + sides:
        s.wait_stream(torch.cuda.current_stream())
    for j in range(args.jobs):
        job(j)
    torch.cuda.synchronize()
    for j, m in enumerate(marks):
        print(f"job {j} s{j % 2}: " + " ".join(f"{k} {t0.elapsed_time(e):7.2f}" for k, e in m.items()))
    for j, h in enumerate(host_t[2:]):
        print(f"job {j} host ms: h2d %.2f from_global %.2f advance %.2f to_global %.2f csum %.2f d2h %.2f" % tuple(h))
    end = max(t0.elapsed_time(m["d2h"]) for m in marks)
    print(f"{end / args.jobs:.2f} ms/job")


if __name__ == "__main__":
    main()
