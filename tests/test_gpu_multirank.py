"""The multi-rank device path end to end on ONE GPU: two processes share
cuda:0 and exchange halos through torch.distributed (gloo, host-staged; with
NCCL the same pack / unpack kernels run around the library's grouped
ncclSend/ncclRecv, tm_halo_exchange, tested here on a one-rank loopback).
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


def worker(rank, world, port, out, fused, shape=(48, 16)):
    import torch.distributed as dist

    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.runner import HeatRunner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # (48, 16): 27 boxes split mid-layer; (48, 8): 216 boxes = three z-layers per rank (the
        # middle one has no remote face); (64, 32): one z-layer of 4 boxes per rank, every box
        # touching the other rank (only their non-boundary planes overlap the exchange)
        w = tm.CONFIGS["C5"].scaled(shape[0], shape[1], 4)  # 2 comps, 2 ghosts
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
            # boundary planes / interior planes as two launches + side stream, also when every box
            # touches the other rank (27 boxes split mid-layer)
            assert r.fh.comm is not None
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


@pytest.mark.parametrize("fused,shape", [(False, (48, 16)), (True, (48, 16)), (True, (48, 8)), (True, (64, 32))])
def test_two_ranks_one_gpu_match_oracle(fused, shape):
    """fused=False: the overlapped unfused step; fused=True: the fused march
    with the remote faces exchanged after each step (slabs: on a side stream,
    overlapping the interior columns' launch)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(2, free_port(), out, fused, shape), nprocs=2, join=True)
    for r in range(2):
        ok, sums_ok, max_ok, min_ok, n = out[r]
        assert ok, f"rank {r}: boxes differ from the oracle"
        assert sums_ok and max_ok and min_ok, f"rank {r}: reductions differ"
    assert out[0][4] + out[1][4] == (shape[0] // shape[1]) ** 3


def nccl_world1_worker(rank, port, out):
    """One NCCL rank: (1) the library's own communicator (tm_comm_create from
    a unique id broadcast over torch.distributed) moves a halo message to
    itself with tm_halo_exchange (grouped ncclSend/ncclRecv), eagerly and
    captured in a CUDA graph; (2) the runner's verified-capture bookkeeping
    (capture pair + eager check pair) lands on the right step."""
    import ctypes

    import torch.distributed as dist

    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200 import _native, halo
    from paper_1604_03570_b200.runner import HeatRunner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        L = _native.load()
        comm = halo.nccl_comm()
        ver = ctypes.c_int32()
        _native.check(L.tm_comm_nccl_version(ctypes.byref(ver)), "version")
        # one "peer" (ourselves): 600 doubles out of sendbuf+100 into recvbuf+50
        pe = np.array([0], np.int32)
        so, sc, ro, rc = (np.array([v], np.int64) for v in (100, 600, 50, 600))
        x = ctypes.c_void_p()
        _native.check(L.tm_exchange_create(comm.handle, 1, pe.ctypes.data, so.ctypes.data, sc.ctypes.data,
                                           ro.ctypes.data, rc.ctypes.data, ctypes.byref(x)), "create")
        src = torch.arange(1000, dtype=torch.float64, device="cuda")
        dst = torch.zeros(700, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        _native.check(L.tm_halo_exchange(x, src.data_ptr(), dst.data_ptr(), st), "eager")
        torch.cuda.synchronize()
        eager_ok = bool(torch.equal(dst[50:650], src[100:700])) and not bool(dst[:50].any())
        dst.zero_()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            src.mul_(2.0)
            _native.check(L.tm_halo_exchange(x, src.data_ptr(), dst.data_ptr(), s.cuda_stream), "captured")
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        a2a_ok = eager_ok and bool(torch.equal(dst[50:650], 2.0 * torch.arange(100, 700, dtype=torch.float64,
                                                                               device="cuda")))
        del g  # a live graph holding NCCL work blocks the communicator's teardown
        L.tm_exchange_destroy(x)
        a2a_ok = a2a_ok and ver.value >= 22000

        w = tm.CONFIGS["C1"].scaled(32, 16, 4)
        geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
        ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
        glob = tm.make_init(w)
        mf = tm.MultiFab(ba, w.ncomp, w.nghost)
        mf.from_global(glob)
        p = tm.HeatParams.stable(1.0, geom.dx)
        r = HeatRunner(mf, geom, p, w.tile_size, fused=True)
        assert r.use_graph
        r._check_graph = True  # what a multi-rank NCCL run does
        r.advance(7)
        got7 = r.current.to_global().cpu().numpy()
        r.advance(5)
        got12 = r.current.to_global().cpu().numpy()
        c = p.coefficients()
        ref7 = orc.heat_periodic(glob, 7, c[:3], c[3])
        ref12 = orc.heat_periodic(ref7, 5, c[:3], c[3])
        out[0] = (a2a_ok, r._graph is not None, bool(np.array_equal(got7, ref7)),
                  bool(np.array_equal(got12, ref12)), r.steps_done)
        r.close()
        halo.close_comm()
    finally:
        dist.destroy_process_group()


def test_nccl_capture_and_verified_replay():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(nccl_world1_worker, args=(free_port(), out), nprocs=1, join=True)
    a2a_ok, kept, ok7, ok12, steps = out[0]
    assert a2a_ok, "tm_halo_exchange loopback (eager or graph-captured) differs"
    assert kept, "verified capture was dropped"
    assert ok7 and ok12, "verified-capture bookkeeping advanced the wrong number of steps"
    assert steps == 12
