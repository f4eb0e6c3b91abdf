"""Timeline of the multi-rank fused step: the boundary planes march, their halo exchange runs on
a side stream while the interior planes march.  Two ranks share cuda:0 through
gloo (host-staged exchange; with NCCL the exchange is tm_halo_exchange), on a layout where
EVERY box touches the other rank (the C2 strong-scaling case at 8 GPUs: 128^3 in 32^3 boxes,
two z-layers per rank, periodic).  Prints, per step and rank, the phase intervals in us from
the step's start (CUDA events on the launching streams).

    python tools/overlap_timeline.py [steps]
"""

import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, steps, out):
    import torch.distributed as dist

    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.runner import HeatRunner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = tm.CONFIGS["C2"].scaled(128, 32, steps)
        geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
        mf = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), 1, 1)
        mf.from_global(tm.make_init(w))
        r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), w.tile_size)
        assert r.fused and r.fh.remote and r.fh.comm is not None
        r.advance(2, finalize=False)  # warm-up
        r.fh.timeline = []
        r.advance(steps, finalize=False)
        torch.cuda.synchronize()
        rows = []
        for m in r.fh.timeline:
            t = {k: m["start"].elapsed_time(e) * 1e3 for k, e in m.items() if k != "start"}
            rows.append(t)
        nb = int(r.fh.plan_b.columns["nz"].sum())
        ni = int(r.fh.plan_i.columns["nz"].sum())
        out[rank] = (rows, nb, ni)
        r.close()
    finally:
        dist.destroy_process_group()


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(2, port, steps, out), nprocs=2, join=True)
    print("C2-like strong-scaling layout: 128^3 in 32^3 boxes over 2 ranks (gloo, one GPU); every box "
          "has a remote face")
    for rank in sorted(out.keys()):
        rows, nb, ni = out[rank]
        print(f"rank {rank}: boundary column-planes {nb}, interior column-planes {ni}")
        for i, t in enumerate(rows):
            ov = max(0.0, min(t["interior_done"], t["exchange_done"]) - max(t["interior_start"], t["exchange_start"]))
            print(f"  step {i}: boundary march 0-{t['boundary_done']:.1f} | interior march "
                  f"{t['interior_start']:.1f}-{t['interior_done']:.1f} | exchange (side stream) "
                  f"{t['exchange_start']:.1f}-{t['exchange_done']:.1f} | overlap {ov:.1f} us")


if __name__ == "__main__":
    main()
