"""Per-rank device time of the peer-halo march on one GPU (emulated ranks) -- the compute part of
a strong-scaled C2 step at N GPUs -- and the device barrier's loopback launch time.

Each emulated rank's march reads its remote faces from the other ranks' storage on the same GPU
(HBM, not NVLink), so this measures the kernel's own time on 1/N of the work: short segments,
more halo planes per interior plane, fewer columns than SMs.  Run: python tools/peer_perf.py
"""

import json
import sys

import torch


def main():
    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.boxarray import DistributionMapping
    from paper_1604_03570_b200.peer import PeerBarrier, PeerFused

    out = {}
    w = tm.CONFIGS["C2"]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    params = tm.HeatParams.stable(1.0, geom.dx)
    glob = torch.randn((1,) + tuple(w.domain.extents[::-1]), dtype=torch.float64, device="cuda")
    for ranks in (1, 2, 4, 8):
        dm = DistributionMapping(ba, ranks)
        pairs = []
        for r in range(ranks):
            a = tm.MultiFab(ba, 1, 1, dm=dm, rank=r)
            a.from_global(glob)
            pairs.append((a, a.clone_empty()))
        fields = {r: (p[0].ptr, p[1].ptr) for r, p in enumerate(pairs)}
        a, b = pairs[0]
        pf = PeerFused(a, b, geom, fields)
        pf.prime(a)
        reps = 200
        for _ in range(10):
            pf.step(b, a, params)
            pf.step(a, b, params, reverse=True)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(reps):
            pf.step(b, a, params)
            pf.step(a, b, params, reverse=True)
        ev[1].record()
        torch.cuda.synchronize()
        us = ev[0].elapsed_time(ev[1]) * 1e3 / (2 * reps)
        # the same steps captured in a graph, with a loopback device barrier before every march
        # (the rank is its own peer: the barrier's device cost without the NVLink round trip)
        bar = PeerBarrier(torch.device("cuda", 0), 0)
        bar.bind([0], [bar.inbox.data_ptr()])
        graph_us = {}
        for with_bar in (False, True):
            pf.barrier = bar if with_bar else None
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g, stream=cs):
                    for _ in range(20):
                        pf.step(b, a, params)
                        pf.step(a, b, params, reverse=True)
            torch.cuda.current_stream().wait_stream(cs)
            g.replay()
            torch.cuda.synchronize()
            ev[0].record()
            for _ in range(10):
                g.replay()
            ev[1].record()
            torch.cuda.synchronize()
            graph_us["with_barrier" if with_bar else "march_only"] = round(ev[0].elapsed_time(ev[1]) * 1e3 / 400, 2)
        pf.barrier = None
        cells = sum(ba[u].ncells for u in a.local_units)
        out[f"C2_strong_{ranks}"] = {"boxes_per_rank": len(a.local_units), "peers": len(pf.peers),
                                     "march_us_per_step_eager": round(us, 2), "graph_us_per_step": graph_us,
                                     "gbs": round(16 * cells / (us * 1e-6) / 1e9, 1)}
        del pairs, pf
    bar = PeerBarrier(torch.device("cuda", 0), 0)
    bar.bind([0], [bar.inbox.data_ptr()])
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(20):
        bar.wait(s)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(1000):
        bar.wait(s)
    ev[1].record()
    torch.cuda.synchronize()
    out["barrier_loopback_eager_us"] = round(ev[0].elapsed_time(ev[1]), 3)  # per 1000 -> us each
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for _ in range(100):
                bar.wait(cs.cuda_stream)
    torch.cuda.current_stream().wait_stream(cs)
    g.replay()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(10):
        g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    out["barrier_loopback_graph_us"] = round(ev[0].elapsed_time(ev[1]), 3)  # per 1000 -> us each
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
