"""The peer (NVLink) halo path on ONE GPU against the single-rank oracle.

* Emulated ranks in one process: every rank's MultiFab pair lives on cuda:0 and
  each rank's march reads its neighbours' faces straight from the other ranks'
  storage (``peer.PeerFused`` with explicit pointers).  The ranks are stepped one
  after another on one stream, which orders them without a barrier (no kernel
  waits on another).  Layouts: the strong-scaled C2 shape at 8 ranks (every box
  has remote y and z faces, 3 peers per rank), slabs with remote z faces only,
  2 components / 2 ghosts (C5 shape), both march directions.
* Two processes sharing cuda:0 through CUDA IPC (``PeerFused.connect``, the
  production setup), ordered by the host barrier (the device barrier is for ranks
  on distinct GPUs), through ``HeatRunner(exchange="peer")``.
* The device barrier on a one-rank loopback (the rank is its own peer), eager and
  inside a captured CUDA graph.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _problem(n, mgs, ncomp, nghost, steps):
    import paper_1604_03570_b200 as tm

    w = tm.CONFIGS["C5"].scaled(n, mgs, steps)
    dom = w.domain
    geom = tm.Geometry(dom, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(dom, mgs)
    rng = np.random.default_rng(7)
    glob = rng.standard_normal((ncomp,) + tuple(dom.extents[::-1]))
    return geom, ba, glob


@pytest.mark.parametrize("n,mgs,ranks,ncomp,nghost", [
    (128, 32, 8, 1, 1),   # C2 strong-scaled shape: 8 boxes per rank, remote y and z faces
    (128, 32, 2, 1, 1),   # slabs: remote z faces only
    (64, 32, 2, 2, 2),    # C5 shape: 2 components, 2 ghosts, one box layer per rank
    (128, 64, 2, 1, 1),   # 64-wide boxes (2 cells per lane)
])
def test_emulated_ranks_match_oracle(n, mgs, ranks, ncomp, nghost):
    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.boxarray import DistributionMapping
    from paper_1604_03570_b200.peer import PeerFused

    steps = 6
    geom, ba, glob = _problem(n, mgs, ncomp, nghost, steps)
    dm = DistributionMapping(ba, ranks)
    pairs = []
    for r in range(ranks):
        a = tm.MultiFab(ba, ncomp, nghost, dm=dm, rank=r)
        a.from_global(glob)
        pairs.append((a, a.clone_empty()))
    fields = {r: (p[0].ptr, p[1].ptr) for r, p in enumerate(pairs)}
    pfs = [PeerFused(a, b, geom, fields) for a, b in pairs]
    assert any(pf.peers for pf in pfs)
    p = tm.HeatParams.stable(1.0, geom.dx)
    for (a, _), pf in zip(pairs, pfs):
        pf.prime(a)
    for k in range(steps):
        for (a, b), pf in zip(pairs, pfs):
            old, new = (a, b) if k % 2 == 0 else (b, a)
            pf.step(new, old, p, reverse=k % 2 == 1)
    torch.cuda.synchronize()
    got = sum(pr[steps % 2].to_global().cpu().numpy() for pr in pairs)
    c = p.coefficients()
    ref = orc.heat_periodic(glob, steps, c[:3], c[3])
    assert np.array_equal(got, ref)


def test_peer_march_rejects_unencoded_set():
    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200 import _native
    from paper_1604_03570_b200.boxarray import DistributionMapping
    from paper_1604_03570_b200.peer import PeerFused

    geom, ba, glob = _problem(64, 32, 1, 1, 1)
    dm = DistributionMapping(ba, 2)
    a0 = tm.MultiFab(ba, 1, 1, dm=dm, rank=0)
    a1 = tm.MultiFab(ba, 1, 1, dm=dm, rank=1)
    pf = PeerFused(a0, a0.clone_empty(), geom, {1: (a1.ptr, a1.ptr)})
    c = tm.HeatParams.stable(1.0, geom.dx).coefficients()
    rc = _native.load().tm_heat_march_peer(pf.plan.handle, a0.layout.to_c(), a0.ptr, pf.b.ptr, 1, c[0], c[1],
                                           c[2], c[3], pf.xh[id(a0)].data_ptr(), pf.xh[id(pf.b)].data_ptr(),
                                           pf.nbr.data_ptr(), 3, 0, a0.stream())
    assert rc == 1 and b"not encoded" in _native.load().tm_last_error()


def test_barrier_loopback_eager_and_graph():
    from paper_1604_03570_b200.peer import PeerBarrier

    bar = PeerBarrier(torch.device("cuda", 0), 0)
    bar.bind([0], [bar.inbox.data_ptr()])  # the rank is its own peer
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        bar.wait(s)
    torch.cuda.synchronize()
    assert int(bar.epoch.item()) == 3 and int(bar.inbox[0].item()) == 3 and not bar.timed_out()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            bar.wait(cs.cuda_stream)
            bar.wait(cs.cuda_stream)
    torch.cuda.current_stream().wait_stream(cs)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    assert int(bar.epoch.item()) == 13 and int(bar.inbox[0].item()) == 13 and not bar.timed_out()


def test_barrier_times_out_instead_of_hanging():
    from paper_1604_03570_b200 import _native
    from paper_1604_03570_b200.peer import PeerBarrier

    bar = PeerBarrier(torch.device("cuda", 0), 0)
    lonely = torch.zeros(_native.MAX_RANKS, dtype=torch.int64, device="cuda")
    bar.bind([1], [lonely.data_ptr()])  # "rank 1" never signals
    _native.check(_native.load().tm_peer_barrier(
        bar.inbox.data_ptr(), bar.peer_inbox.data_ptr(), bar.peer_ranks.data_ptr(), 1, 0, bar.epoch.data_ptr(),
        bar.status.data_ptr(), 20_000_000, torch.cuda.current_stream().cuda_stream), "barrier")
    torch.cuda.synchronize()
    assert bar.timed_out() and int(lonely[0].item()) == 1


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, out, n, mgs, ncomp=1, nghost=1):
    import torch.distributed as dist

    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.runner import HeatRunner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        steps = 7
        geom, ba, glob = _problem(n, mgs, ncomp, nghost, steps)
        mf = tm.MultiFab(ba, ncomp, nghost)
        mf.from_global(glob)
        p = tm.HeatParams.stable(1.0, geom.dx)
        r = HeatRunner(mf, geom, p, fused=True, exchange="peer")
        assert r.exchange == "peer" and r.fh.host_barrier and r.fh.peers and not r.use_graph
        fin = r.advance(steps)
        got = fin.to_global().cpu().numpy()
        c = p.coefficients()
        ref = orc.heat_periodic(glob, steps, c[:3], c[3])
        mine = np.zeros_like(ref)
        for u in fin.local_units:
            v = ba[u]
            sl = (slice(None),) + tuple(slice(v.lo[d], v.hi[d] + 1) for d in (2, 1, 0))
            mine[sl] = ref[sl]
        h = orc.HostMF(list(ba), ncomp, nghost)
        h.from_global(ref)
        out[rank] = (bool(np.array_equal(got, mine)),
                     all(fin.reduce_sum(k) == orc.reduce_sum(h, k) for k in range(ncomp)))
        torch.cuda.synchronize()
        dist.barrier()
        r.fh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,mgs,world,ncomp,nghost", [(64, 32, 2, 1, 1), (128, 32, 2, 1, 1), (64, 32, 2, 2, 2),
                                                       (128, 32, 4, 1, 1)])
def test_two_processes_ipc_match_oracle(n, mgs, world, ncomp, nghost):
    """Real CUDA IPC between processes sharing cuda:0 (2 ranks; 4 ranks: every box has remote
    z faces on two different peers)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(world, free_port(), out, n, mgs, ncomp, nghost), nprocs=world, join=True)
    for r in range(world):
        ok, sum_ok = out[r]
        assert ok, f"rank {r}: boxes differ from the oracle"
        assert sum_ok, f"rank {r}: checksum differs"
