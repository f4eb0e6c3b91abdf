"""The multi-rank device path end to end on ONE GPU: two processes share
cuda:0 and exchange halos through torch.distributed (gloo, host-staged; the
bench uses NCCL over NVLink with the same pack / send-recv / unpack code).
No kernel waits on another process, so sharing the device is safe.  Checks
the overlapped step (interior sweep while messages are in flight), the fused
march with its cross-rank face exchange, the multi-rank checksum protocol and
max/min against the single-rank oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, out, fused):
    import torch.distributed as dist

    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.runner import HeatRunner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = tm.CONFIGS["C5"].scaled(48, 16, 4)  # 27 boxes, 2 comps, 2 ghosts
        geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
        ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
        glob = tm.make_init(w)
        mf = tm.MultiFab(ba, w.ncomp, w.nghost)  # DistributionMapping over the gloo world
        mf.from_global(glob)
        p = tm.HeatParams.stable(1.0, geom.dx)
        r = HeatRunner(mf, geom, p, w.tile_size, fused=fused)
        assert r.fused == fused and not r.use_graph
        if fused:  # the 27 boxes split mid-layer: remote neighbours in x, y and z
            assert r.fh.remote
        fin = r.advance(w.steps)
        got = fin.to_global().cpu().numpy()  # only this rank's boxes are non-zero
        c = p.coefficients()
        ref = orc.heat_periodic(glob, w.steps, c[:3], c[3])
        mine = np.zeros_like(ref)
        for u in fin.local_units:
            v = ba[u]
            sl = (slice(None),) + tuple(slice(v.lo[d], v.hi[d] + 1) for d in (2, 1, 0))
            mine[sl] = ref[sl]
        h = orc.HostMF(list(ba), w.ncomp, w.nghost)
        h.from_global(ref)
        sums = [fin.reduce_sum(k) for k in range(w.ncomp)]
        out[rank] = (bool(np.array_equal(got, mine)), sums == [orc.reduce_sum(h, k) for k in range(w.ncomp)],
                     fin.reduce_max(1) == orc.reduce_max(h, 1), fin.reduce_min(0) == orc.reduce_min(h, 0),
                     len(fin.local_units))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
def test_two_ranks_one_gpu_match_oracle(fused):
    """fused=False: the overlapped unfused step; fused=True: the fused march
    with the remote faces exchanged after each step."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(2, free_port(), out, fused), nprocs=2, join=True)
    for r in range(2):
        ok, sums_ok, max_ok, min_ok, n = out[r]
        assert ok, f"rank {r}: boxes differ from the oracle"
        assert sums_ok and max_ok and min_ok, f"rank {r}: reductions differ"
    assert out[0][4] + out[1][4] == 27
