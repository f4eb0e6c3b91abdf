"""Inter-GPU FillBoundary: packed halo messages over NCCL.

The reference is single-process and has no exchange; the
multi-GPU path is new.  Each rank holds the global
FillBoundary plan (identical on every rank: it is a pure function of the
BoxArray, geometry and ghost width) and the DistributionMapping, so both
ends of every message derive the same layout without any metadata
exchange:

* the message from rank a to rank b is the ordered list of plan tags whose
  source unit a owns and whose destination unit b owns, each tag's cells
  packed x-fastest then y, z, component (``tm_side`` "packed" format);
* rank a packs all its outgoing messages with one copy-kernel launch into
  one send buffer (messages in ascending peer order), every message of the
  exchange travels in ONE grouped ``ncclSend`` / ``ncclRecv`` with the
  neighbour ranks only (``tm_halo_exchange`` in the C-ABI, on the library's
  own communicator: torch.distributed only carries the unique id at setup),
  and rank b unpacks all its incoming messages with one launch straight
  into ghost cells.  One host call per exchange keeps the issue cost low,
  and the exchange is capturable in a CUDA graph (``runner.HeatRunner``
  replays multi-rank steps).  Under the gloo backend (CPU tests, several
  ranks sharing one GPU) the messages go through a host-staged
  ``all_to_all_single`` with per-peer split sizes instead.

Intra-rank tags never touch a buffer: they are the local copy kernel.
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np

from . import _native


def exchange_lists(owners, tags, me: int):
    """Split plan tag indices for rank ``me``:
    ``(local, sends{peer: [tag ids]}, recvs{peer: [tag ids]})``; peers in
    ascending rank order, tag ids in plan order on both ends."""
    local = []
    sends: dict = {}
    recvs: dict = {}
    for n, t in enumerate(tags):
        so, do = owners[t[2]], owners[t[0]]
        if so == me and do == me:
            local.append(n)
        elif so == me:
            sends.setdefault(do, []).append(n)
        elif do == me:
            recvs.setdefault(so, []).append(n)
    return (local, OrderedDict(sorted(sends.items())), OrderedDict(sorted(recvs.items())))


def tag_elements(tag, ncomp: int) -> int:
    e = tag[1].extents
    return e[0] * e[1] * e[2] * ncomp


def message_layout(tags, groups, ncomp: int):
    """Packed buffer layout of the messages in ``groups`` ({peer: [tag ids]}):
    ``(rows, spans, total)`` with rows = [(tag id, element offset)] in buffer
    order and spans = [(peer, offset, count)].  Inside a tag the elements are
    x fastest, then y, z, component (the ``tm_side`` packed format)."""
    rows, spans, off = [], [], 0
    for peer, ids in groups.items():
        start = off
        for n in ids:
            rows.append((n, off))
            off += tag_elements(tags[n], ncomp)
        spans.append((peer, start, off - start))
    return rows, spans, off


def split_sizes(spans, world: int) -> list:
    """Per-rank element counts of a message buffer for
    ``all_to_all_single``: spans' counts at their peers, 0 elsewhere (self
    included).  Valid because ``message_layout`` orders messages by
    ascending peer."""
    sizes = [0] * world
    for peer, _, n in spans:
        sizes[peer] = n
    return sizes


class HaloExchange:
    """Pack / grouped send-recv / unpack for one (MultiFab layout, plan)."""

    def __init__(self, mf, plan):
        import torch

        from .multifab import cell_offsets

        self.device = mf.device
        tags = plan.tags
        _, sends, recvs = exchange_lists(mf.unit_owner, tags, mf.rank)
        nc = mf.ncomp

        def build(groups, remote_side_is_dst):
            layout, spans, off = message_layout(tags, groups, nc)
            rows = [(tags[n], o, tags[n][1].extents) for n, o in layout]
            arr = np.zeros(len(rows), dtype=_native.COPY_TAG_DTYPE)
            if rows:
                units = np.array([r[0][2] if remote_side_is_dst else r[0][0] for r in rows], dtype=np.int64)
                cells = np.array([r[0][3].lo if remote_side_is_dst else r[0][1].lo for r in rows], dtype=np.int64)
                field = cell_offsets(mf, units, cells)
                buf = np.array([r[1] for r in rows], dtype=np.int64)
                ext = np.array([r[2] for r in rows], dtype=np.int64)
                if remote_side_is_dst:  # pack: storage -> send buffer
                    arr["dst_off"], arr["src_off"] = buf, field
                else:  # unpack: receive buffer -> storage
                    arr["dst_off"], arr["src_off"] = field, buf
                arr["ex"], arr["ey"], arr["ez"] = ext[:, 0], ext[:, 1], ext[:, 2]
            return arr, spans, off

        # ghost boxes of local units that only a remote rank can fill (for overlap splitting)
        self.remote_dst: dict = {}
        for ids in recvs.values():
            for n in ids:
                self.remote_dst.setdefault(tags[n][0], []).append(tags[n][1])
        # local units whose valid cells some other rank needs, and those cells (source boxes)
        self.send_src: dict = {}
        for ids in sends.values():
            for n in ids:
                self.send_src.setdefault(tags[n][2], []).append(tags[n][3])
        self.send_units = sorted(self.send_src)
        pack_tags, self.send_spans, nsend = build(sends, True)
        unpack_tags, self.recv_spans, nrecv = build(recvs, False)
        self.pack = _native.CopyPlan(pack_tags, nc)
        self.unpack = _native.CopyPlan(unpack_tags, nc)
        self.sendbuf = torch.empty(max(nsend, 1), dtype=torch.float64, device=mf.device)
        self.recvbuf = torch.empty(max(nrecv, 1), dtype=torch.float64, device=mf.device)
        self.bytes_sent = nsend * 8
        self.bytes_recv = nrecv * 8
        self.nsend, self.nrecv = nsend, nrecv
        self.send_splits = split_sizes(self.send_spans, mf.dm.nranks)
        self.recv_splits = split_sizes(self.recv_spans, mf.dm.nranks)
        self._work = None
        self._host = None
        self._side = None  # NCCL: pack + send/recv run on this stream
        self._x = None     # NCCL: tm_exchange handle

    def start(self, mf, stream: int) -> None:
        """Pack every outgoing message of ``mf`` (one launch) and post the
        exchange.  Over NCCL both go on this exchange's side stream (forked
        from the current stream), so work the caller queues next overlaps the
        transfer; ``finish`` joins the side stream and unpacks.  The exchange
        object is shared by every MultiFab of the same layout (e.g. both
        buffers of a double-buffered pair), so the field is passed per call."""
        import torch

        if self._host is None:
            import torch.distributed as dist

            self._host = dist.get_backend() == "gloo"
        if self._host:  # CPU transport (tests): stage through host memory, torch all-to-all
            import torch.distributed as dist

            self.pack.run(self.sendbuf.data_ptr(), (0, 0, 0), mf.ptr, mf.layout.side(), stream)
            torch.cuda.current_stream(self.device).synchronize()
            sbuf = self.sendbuf[:self.nsend].cpu()
            self._hrecv = torch.empty(self.nrecv, dtype=torch.float64)
            self._work = dist.all_to_all_single(self._hrecv, sbuf, self.recv_splits, self.send_splits,
                                                async_op=True)
            return
        x = self._nccl_exchange()
        cur = torch.cuda.current_stream(self.device)
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
        self._side.wait_stream(cur)
        side = self._side.cuda_stream
        self.pack.run(self.sendbuf.data_ptr(), (0, 0, 0), mf.ptr, mf.layout.side(), side)
        _native.check(_native.load().tm_halo_exchange(x, self.sendbuf.data_ptr(), self.recvbuf.data_ptr(), side),
                      "tm_halo_exchange")

    def finish(self, mf, stream: int) -> None:
        import torch

        if self._host:
            if self._work is not None:
                self._work.wait()
            self._work = None
            self.recvbuf[:self.nrecv].copy_(self._hrecv)
        else:
            torch.cuda.current_stream(self.device).wait_stream(self._side)
        self.unpack.run(mf.gptr, mf.layout.side(), self.recvbuf.data_ptr(), (0, 0, 0), stream)

    def _nccl_exchange(self):
        """The library-side plan of this exchange's messages (``tm_exchange``:
        neighbour ranks only, offsets into the send / receive buffers)."""
        if self._x is None:
            import ctypes

            peers = sorted({p for p, _, n in self.send_spans if n} | {p for p, _, n in self.recv_spans if n})
            send = {p: (o, n) for p, o, n in self.send_spans}
            recv = {p: (o, n) for p, o, n in self.recv_spans}
            arr = lambda v, t: np.ascontiguousarray(np.array(v, dtype=t).reshape(-1))  # noqa: E731
            pe = arr(peers, np.int32)
            so = arr([send.get(p, (0, 0))[0] for p in peers], np.int64)
            sc = arr([send.get(p, (0, 0))[1] for p in peers], np.int64)
            ro = arr([recv.get(p, (0, 0))[0] for p in peers], np.int64)
            rc = arr([recv.get(p, (0, 0))[1] for p in peers], np.int64)
            h = ctypes.c_void_p()
            ptr = lambda a: a.ctypes.data if len(a) else None  # noqa: E731
            _native.check(_native.load().tm_exchange_create(nccl_comm().handle, len(peers), ptr(pe), ptr(so),
                                                            ptr(sc), ptr(ro), ptr(rc), ctypes.byref(h)),
                          "tm_exchange_create")
            self._x = h
            self._keep = (pe, so, sc, ro, rc)
            self.peers = peers
        return self._x

    def __del__(self):
        x = getattr(self, "_x", None)
        if x is not None and _native._lib is not None:
            _native._lib.tm_exchange_destroy(x)
            self._x = None


class NcclComm:
    """The process's NCCL communicator for halo traffic (``tm_comm``), built
    once over the default torch.distributed group: rank 0's unique id is
    broadcast through torch.distributed at setup only; every message after
    that goes through the library (``tm_halo_exchange``)."""

    def __init__(self):
        import ctypes

        import torch.distributed as dist

        L = _native.load()
        rank, world = dist.get_rank(), dist.get_world_size()
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _native.check(L.tm_comm_unique_id(uid), "tm_comm_unique_id")
        box = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        h = ctypes.c_void_p()
        _native.check(L.tm_comm_create(box[0], world, rank, ctypes.byref(h)), "tm_comm_create")
        self.handle = h
        self.rank, self.world = rank, world

    def close(self) -> None:
        if self.handle is not None and _native._lib is not None:
            _native._lib.tm_comm_destroy(self.handle)
        self.handle = None


_COMM = None


def nccl_comm() -> NcclComm:
    global _COMM
    if _COMM is None:
        _COMM = NcclComm()
    return _COMM


def close_comm() -> None:
    """Destroy the halo communicator (before ``destroy_process_group``; any
    graph holding its work must be released first)."""
    global _COMM
    if _COMM is not None:
        _COMM.close()
        _COMM = None
