"""Multi-rank FillBoundary protocol on CPU (gloo, world size 2 and 3).

Each rank owns the boxes DistributionMapping assigns it, derives its local /
send / receive tag lists and packed message layouts from the GLOBAL plan
(``halo.exchange_lists`` + ``halo.message_layout`` -- the same functions the
GPU HaloExchange uses), packs its outgoing tags with numpy, exchanges the
messages with one ``all_to_all_single`` (per-peer split sizes, as the
device HaloExchange does) and unpacks.  The ghosts of every box a
rank owns must equal the single-process oracle FillBoundary bit for bit.
Also checks the multi-rank checksum protocol (partials all-reduced, then
summed in grid order) against the serial reference sum.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1604_03570_b200 import Box, BoxArray, DistributionMapping, Geometry
from paper_1604_03570_b200.fillplan import build_fill_plan_units
from paper_1604_03570_b200.halo import exchange_lists, message_layout, split_sizes

NC, NG = 2, 2


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def layout():
    dom = Box((0, 0, 0), (23, 15, 19))
    ba = BoxArray.chop(dom, (8, 8, 5))  # 3 x 2 x 4 = 24 boxes, uneven z
    geom = Geometry(dom, (True, True, False))
    return dom, list(ba), geom


def field(n):
    rng = np.random.default_rng(123)
    return rng.random((NC,) + tuple(n))


def tag_region(h, t, src: bool):
    """numpy view (nx, ny, nz, nc) of a tag's src or dst box in HostMF h."""
    u = t.src_unit if src else t.dst_unit
    b = t.src_box if src else t.dst_box
    lo = h.lo[u]
    sl = tuple(slice(b.lo[d] - lo[d], b.hi[d] - lo[d] + 1) for d in range(3))
    return h.fab(u)[sl]


def pack(h, tags, rows, total):
    buf = np.empty(total)
    for n, off in rows:
        blk = tag_region(h, tags[n], True)
        # packed order: x fastest, then y, z, component
        buf[off:off + blk.size] = blk.ravel(order="F")
    return buf


def unpack(h, tags, rows, buf):
    for n, off in rows:
        view = tag_region(h, tags[n], False)
        view[...] = buf[off:off + view.size].reshape(view.shape, order="F")


def worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dom, valids, geom = layout()
        plan = build_fill_plan_units(valids, geom, NG, grids=valids)
        dm = DistributionMapping(len(valids), world)
        local, sends, recvs = exchange_lists(dm.owners, plan.tags, rank)
        glob = field(tuple(reversed(dom.extents)))
        h = orc.HostMF(valids, NC, NG, fill=np.nan)
        h.from_global(glob)
        for u in range(len(valids)):  # this rank only has its own boxes
            if dm[u] != rank:
                h.fab(u)[...] = np.nan
        orc.fill_boundary(h, [plan.tags[n] for n in local])
        srows, sspans, stot = message_layout(plan.tags, sends, NC)
        rrows, rspans, rtot = message_layout(plan.tags, recvs, NC)
        sendbuf = torch.from_numpy(pack(h, plan.tags, srows, stot))
        recvbuf = torch.empty(rtot, dtype=torch.float64)
        assert [o for _, o, _ in sspans] == sorted(o for _, o, _ in sspans)  # ascending peers
        dist.all_to_all_single(recvbuf, sendbuf, split_sizes(rspans, world), split_sizes(sspans, world))
        unpack(h, plan.tags, rrows, recvbuf.numpy())
        ref = orc.HostMF(valids, NC, NG, fill=np.nan)
        ref.from_global(glob)
        orc.fill_boundary(ref, plan.tags)
        ok = all(np.array_equal(h.fab(u), ref.fab(u), equal_nan=True) for u in range(len(valids)) if dm[u] == rank)
        # checksum protocol: one contributor per partial, then grid-order serial sum
        part = torch.zeros(len(valids), dtype=torch.float64)
        for u in range(len(valids)):
            if dm[u] == rank:
                v = h.valid_view(u, 0)
                s = 0.0
                for x in np.ravel(v, order="F"):
                    s += x
                part[u] = s
        dist.all_reduce(part)
        total = 0.0
        for x in part.tolist():
            total += x
        out[rank] = (ok, total == orc.reduce_sum(ref, 0), stot, rtot)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_fill_boundary_gloo(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(world, free_port(), out), nprocs=world, join=True)
    assert len(out) == world
    for r in range(world):
        ok, sum_ok, sent, recvd = out[r]
        assert ok, f"rank {r} ghosts differ from the single-process fill"
        assert sum_ok, f"rank {r} checksum protocol differs from the serial sum"
        assert sent > 0 and recvd > 0
    assert sum(out[r][2] for r in range(world)) == sum(out[r][3] for r in range(world))


def test_exchange_lists_partition_every_tag():
    dom, valids, geom = layout()
    plan = build_fill_plan_units(valids, geom, NG, grids=valids)
    for world in (1, 2, 3, 5):
        dm = DistributionMapping(len(valids), world)
        seen = []
        for r in range(world):
            local, sends, recvs = exchange_lists(dm.owners, plan.tags, r)
            seen += local
            for p, ids in recvs.items():
                # what r receives from p is exactly what p sends to r, same order
                _, psends, _ = exchange_lists(dm.owners, plan.tags, p)
                assert psends[r] == ids
                seen += ids
        assert sorted(seen) == list(range(len(plan.tags)))
