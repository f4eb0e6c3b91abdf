"""Peer (NVLink / NVSwitch) halos: the FillBoundary exchange fused into the sweep.

The reference's seam is ``fill_boundary`` (``/root/reference/pkg/src/tilemesh/level.py:297-323``)
followed by ``heat_step`` (``kernels.py:174-215``).  With boxes on several GPUs the remote part
of the fill is, in the NCCL path (``halo.py``), a pack launch, a grouped send/recv and an unpack
launch per step.  Here the step's march kernel (``tm_heat_march_peer``, TM_HALO_FUSED_NBR) TMA-
loads every y/z halo plane and row whose face neighbour lives on another rank straight from
that rank's valid cells over NVLink while it computes -- no pack, no message, no unpack, no
ghost writes -- and one ``tm_peer_barrier`` launch between steps orders the ranks.  BoxLib's
aggregated remote ghost traffic it replaces: ``/root/reference/PAPER.md:549-556``.

Rules (checked here): every face is covered by exactly one box of the same extents
(``march.fusable``), the x faces of every local box are local (the packed x halos are written by
the local epilogue), columns are of one height and a width that is a multiple of 16 (the
neighbour-halo march), at most ``MAX_PEERS`` peer ranks, and every rank shares the storage
layout apart from its slot count.

Two ways to connect the peers' storage:

* ``PeerFused.connect`` (collective over ``torch.distributed``): every rank exports CUDA IPC
  handles of its two fields and of its barrier inbox (``tm_ipc_export``), all-gathers them, and
  maps the handles of the ranks it neighbours (``tm_ipc_open``).  Steps are ordered by the device
  barrier (ranks on distinct GPUs) or, with ``barrier="host"`` (ranks sharing one GPU, tests),
  by the caller synchronising between steps.
* ``PeerFused(..., peer_fields={rank: (ptr_a, ptr_b)})``: explicit pointers -- several ranks'
  MultiFabs in one process (the single-GPU emulation the tests use; the caller steps the ranks
  one after another, which orders them without a barrier).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .boxarray import Geometry
from .march import (REMOTE, default_fused_rows, face_neighbors, fusable, march_plan, xh_init_plan)
from .multifab import MultiFab

BARRIER_TIMEOUT_NS = 10_000_000_000  # a peer that never arrives: status flag after 10 s, no hang


def _slots_by_rank(mf: MultiFab) -> dict:
    """rank -> its local units in slot order (every rank derives every rank's slots)."""
    out: dict = {}
    for u, r in enumerate(mf.unit_owner):
        out.setdefault(r, []).append(u)
    return out


def peer_face_table(mf: MultiFab, geom: Geometry):
    """(table, peer_ranks): per local slot the 6 face entries (-x,+x,-y,+y,-z,+z) with faces on
    another rank encoded ``TM_NBR_PEER(p, s)`` (slot s of ``peer_ranks[p]``).  Raises
    ValueError when the layout cannot take the peer path."""
    if not fusable(mf, geom, allow_remote=True):
        raise ValueError("peer halos need a uniform fully-covered box layout (march.fusable)")
    table = face_neighbors(mf, geom, allow_remote=True).copy()
    if not (table[:, :2] != REMOTE).all():
        raise ValueError("peer halos need every x-face neighbour on the same rank (packed x halos are local)")
    by_rank = _slots_by_rank(mf)
    slot_on = {r: {u: s for s, u in enumerate(us)} for r, us in by_rank.items()}
    # the remote neighbour's unit: the box that covers the face image (face_neighbors' rule)
    from .box import Box
    from .boxarray import BoxIndex

    valids = [u.valid for u in mf.units]
    index = BoxIndex(valids)
    dom, n = geom.domain, geom.domain.extents
    peers: list = []
    for s, u in enumerate(mf.local_units):
        v = valids[u]
        e = v.extents
        for k in range(2, 6):
            if table[s, k] != REMOTE:
                continue
            d, side = divmod(k, 2)
            lo = list(v.lo)
            lo[d] += -e[d] if side == 0 else e[d]
            lo[d] = dom.lo[d] + (lo[d] - dom.lo[d]) % n[d]
            nb = index.query(Box(lo, [lo[i] + e[i] - 1 for i in range(3)]))[0]
            r = mf.unit_owner[nb]
            if r not in peers:
                peers.append(r)
            table[s, k] = _native.nbr_peer(peers.index(r), slot_on[r][nb])
    if len(peers) > _native.MAX_PEERS:
        raise ValueError(f"peer halos: {len(peers)} peer ranks > {_native.MAX_PEERS}")
    return table, peers


class PeerBarrier:
    """Device barrier between this rank and its peer ranks (``tm_peer_barrier``): an inbox of
    ``MAX_RANKS`` counters in this rank's memory, written by the peers through IPC."""

    def __init__(self, device, rank: int):
        import torch

        self.rank = rank
        self.inbox = torch.zeros(_native.MAX_RANKS, dtype=torch.int64, device=device)
        self.epoch = torch.zeros(1, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.peer_ranks = None
        self.peer_inbox = None
        self.npeers = 0

    def bind(self, peer_ranks: list, inbox_ptrs: list) -> None:
        import torch

        dev = self.inbox.device
        self.npeers = len(peer_ranks)
        self.peer_ranks = torch.as_tensor(np.array(peer_ranks, dtype=np.int32), device=dev)
        self.peer_inbox = torch.as_tensor(np.array(inbox_ptrs, dtype=np.int64), device=dev)

    def wait(self, stream: int) -> None:
        if self.npeers == 0:
            return
        _native.check(_native.load().tm_peer_barrier(
            self.inbox.data_ptr(), self.peer_inbox.data_ptr(), self.peer_ranks.data_ptr(), self.npeers, self.rank,
            self.epoch.data_ptr(), self.status.data_ptr(), BARRIER_TIMEOUT_NS, stream), "tm_peer_barrier")

    def timed_out(self) -> bool:
        return bool(self.status.item())


def ipc_export(ptr: int) -> tuple:
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _native.check(_native.load().tm_ipc_export(ptr, h, ctypes.byref(off)), "tm_ipc_export")
    return h.raw, off.value


def ipc_open(handle: bytes, offset: int) -> int:
    p = ctypes.c_void_p(0)
    _native.check(_native.load().tm_ipc_open(handle, offset, ctypes.byref(p)), "tm_ipc_open")
    return p.value


class PeerFused:
    """The fused march of a double-buffered pair (a, b) with faces on other ranks read from the
    peers' storage.  ``step`` has the signature of ``march.FusedHalo.step``."""

    def __init__(self, a: MultiFab, b: MultiFab, geom: Geometry, peer_fields: dict,
                 max_rows: int | None = None, nctas: int | None = None, barrier: PeerBarrier | None = None):
        import torch

        if not a.same_layout(b):
            raise ValueError("peer halos: the pair must share one layout")
        self.geom, self.a, self.b = geom, a, b
        self.table, self.peers = peer_face_table(a, geom)
        missing = [r for r in self.peers if r not in peer_fields]
        if missing:
            raise ValueError(f"peer halos: no storage for peer ranks {missing}")
        L = a.layout
        self.nyv = L.ny - 2 * L.nghost
        self.nzv = L.nz - 2 * L.nghost
        shape = (L.nslots * a.ncomp, self.nzv, 2, self.nyv)
        self.xh = {id(a): torch.zeros(shape, dtype=torch.float64, device=a.device),
                   id(b): torch.zeros(shape, dtype=torch.float64, device=a.device)}
        self.nbr = torch.as_tensor(self.table.reshape(-1), dtype=torch.int32, device=a.device)
        self.plan = march_plan(a, True, max_rows if max_rows is not None else default_fused_rows(a), nctas)
        cols = self.plan.columns
        if len(set(cols["ny"].tolist())) != 1 or int(cols["nx"].max()) % 16:
            raise ValueError("peer halos need the neighbour-halo march (columns of one height, width % 16 == 0)")
        by_rank = _slots_by_rank(a)
        nslots = (ctypes.c_int64 * max(1, len(self.peers)))(*[len(by_rank[r]) for r in self.peers])
        lib = _native.load()
        for field in (0, 1):
            bases = (ctypes.c_void_p * max(1, len(self.peers)))(*[peer_fields[r][field] for r in self.peers])
            _native.check(lib.tm_march_plan_set_peers(self.plan.handle, field, a.layout.to_c(), len(self.peers),
                                                      bases, nslots), "tm_march_plan_set_peers")
        self._init, self.xh_side = xh_init_plan(a, self.table, self.nyv, self.nzv)
        self.barrier = barrier
        self.host_group = None  # connect(barrier="host"): the process group the host barrier uses
        self.host_barrier = False
        self.mode = _native.HALO_FUSED_NBR
        self.remote = False  # no exchange after the step: the march reads the peers itself
        self._opened: list = []

    @classmethod
    def connect(cls, a: MultiFab, b: MultiFab, geom: Geometry, barrier: str = "device", group=None,
                max_rows: int | None = None, nctas: int | None = None) -> "PeerFused":
        """Collective: exchange IPC handles of every rank's pair (and barrier inbox) and build
        this rank's peer march.  ``barrier="device"``: ``tm_peer_barrier`` orders the steps
        (ranks on distinct GPUs); ``"host"``: the caller orders them (ranks sharing a GPU)."""
        import torch.distributed as dist

        rank = dist.get_rank(group)
        bar = PeerBarrier(a.device, rank) if barrier == "device" else None
        mine = {"rank": rank, "a": ipc_export(a.ptr), "b": ipc_export(b.ptr),
                "inbox": ipc_export(bar.inbox.data_ptr()) if bar is not None else None,
                "layout": tuple(a.layout)[1:], "device": torch_device_uuid(a.device)}
        every: list = [None] * dist.get_world_size(group)
        dist.all_gather_object(every, mine, group=group)
        _, peers = peer_face_table(a, geom)
        # one mapping per exported allocation: a peer's fields (and inbox) may share one
        # caching-allocator segment, i.e. one IPC handle at different offsets
        bases: dict = {}

        def open_(h):
            handle, off = h
            if handle not in bases:
                bases[handle] = ipc_open(handle, 0)
            return bases[handle] + off

        fields = {}
        for r in peers:
            e = every[r]
            if e["layout"] != mine["layout"]:
                raise ValueError(f"peer halos: rank {r} has another storage layout")
            fields[r] = (open_(e["a"]), open_(e["b"]))
        self = cls(a, b, geom, fields, max_rows, nctas)
        if bar is not None:
            bar.bind(self.peers, [open_(every[r]["inbox"]) for r in self.peers])
            self.barrier = bar
        else:
            self.host_barrier, self.host_group = True, group
        self._opened = [(p, 0) for p in bases.values()]
        return self

    def close(self) -> None:
        lib = _native.load()
        for p, off in self._opened:
            lib.tm_ipc_close(p, off)
        self._opened = []

    def prime(self, mf: MultiFab, plan=None) -> None:
        """Packed x halos of ``mf`` from its local x neighbours' valid cells (the y/z halos are
        read from the neighbours themselves by every step: no ghost fill is needed)."""
        self._init.run(self.xh[id(mf)].data_ptr(), self.xh_side, mf.ptr, mf.layout.side(), mf.stream())

    def step(self, new: MultiFab, old: MultiFab, params, reverse: bool = False) -> None:
        """One step old -> new: barrier with the peers (device mode), then one march launch whose
        TMA producer reads peer faces from peer set 0 (old is ``a``) or 1 (old is ``b``)."""
        if old is self.a:
            field = 0
        elif old is self.b:
            field = 1
        else:
            raise ValueError("peer step: old must be one of the pair")
        s = old.stream()
        if self.barrier is not None:
            self.barrier.wait(s)
        elif self.host_barrier:  # ranks sharing a GPU: every rank's previous step is complete
            import torch
            import torch.distributed as dist

            torch.cuda.synchronize(old.device)
            dist.barrier(group=self.host_group)
        c = params.coefficients()
        _native.check(_native.load().tm_heat_march_peer(
            self.plan.handle, old.layout.to_c(), old.ptr, new.wgptr, old.ncomp, c[0], c[1], c[2], c[3],
            self.xh[id(old)].data_ptr(), self.xh[id(new)].data_ptr(), self.nbr.data_ptr(), field, int(reverse), s),
            "tm_heat_march_peer")


def torch_device_uuid(device) -> str:
    import torch

    try:
        return str(torch.cuda.get_device_properties(device).uuid)
    except Exception:  # pragma: no cover
        return ""


def ranks_share_device(device) -> bool:
    """Collective: True when two ranks of the default group run on the same physical GPU (the
    device barrier must then not be used: kernels that wait on one another cannot share a GPU)."""
    import torch.distributed as dist

    every: list = [None] * dist.get_world_size()
    dist.all_gather_object(every, torch_device_uuid(device))
    return len(set(every)) < len(every) or "" in every
