"""Step loops: ``steps x (FillBoundary; sweep)`` captured as CUDA graphs.

The reference's driver loop (bench.py:198-206) calls ``fill_boundary`` and
``heat_step`` from Python every step.  On the GPU a step of config C2 is
tens of microseconds of device time, comparable to the Python + ctypes cost
of issuing it, so ``HeatRunner`` captures a double-buffered pair of steps
(old -> new, new -> old) once into a CUDA graph and replays it.  Every launch
inside the graph is a library kernel with arguments (and TMA descriptors)
frozen at capture time; the buffers never move, so replay is exact.

Two step implementations, bit-identical in the valid cells:

* ``fused=False`` -- the reference's structure: FillBoundary (Kernel B)
  then the tiled sweep (Kernel A), two launches per step;
* ``fused=True``  -- one launch per step: the persistent column-march sweep
  reads face halos that the previous step's epilogue wrote and scatters its
  own boundary values into the neighbours' halos (``march.FusedHalo``).
  Edge/corner ghosts (unused by the 7-point stencil) are refreshed by one
  regular FillBoundary at the end of ``advance``, so the MultiFab handed
  back has every ghost filled.

Multi-rank, ``exchange="peer"``: the march reads the faces of boxes on other
ranks straight from their storage over NVLink (``peer.PeerFused``), one
device barrier launch between steps; no pack, message or unpack.

Multi-rank: fused, the march scatters into local neighbours and the faces
shared with other ranks travel as one packed all-to-all (NCCL) of the new
field right after it; unfused, the interior tiles are swept while the halo
messages are in flight (``stencil.overlapped_step``).  Over NCCL the step
pair -- kernels and collectives -- is captured into the graph too, so a step
costs no Python; the first captured pair is checked bit for bit against two
eager steps on every rank (all-reduced verdict), and the runner falls back to
eager steps if any rank disagrees.  ``TM_MULTI_GRAPH=0`` forces eager steps.
"""

from __future__ import annotations

import os

from .boxarray import Geometry
from .fillplan import FillPlan, build_fill_plan
from .mfiter import TileSchedule, build_schedule
from .multifab import MultiFab, comm_info, fill_boundary
from .stencil import HeatParams, heat_step, overlapped_step


class HeatRunner:
    """Owns the old/new pair and advances it ``n`` steps at a time."""

    LONG_PAIRS = 8  # captured pairs per replay of the long graph (one rank)

    def __init__(self, mf: MultiFab, geom: Geometry, params: HeatParams, schedule=None,
                 plan: FillPlan | None = None, use_graph: bool | None = None, zmerge: bool = False,
                 fused: bool | None = None, march_rows: int | None = None, exchange: str = "nccl"):
        from . import march

        self.geom = geom
        self.params = params
        self.a = mf
        self.b = mf.clone_empty()
        self.plan = plan if plan is not None else build_fill_plan(mf, geom)
        if schedule is None or not isinstance(schedule, TileSchedule):
            schedule = build_schedule(mf, "default" if schedule is None else schedule)
        self.schedule = schedule
        self.zmerge = zmerge
        world = comm_info()[1]
        graphable = world == 1 or _nccl_world()
        self.use_graph = graphable if use_graph is None else (use_graph and graphable)
        self._check_graph = world > 1
        can_fuse = march.fusable(mf, geom, allow_remote=world > 1)
        if fused and not can_fuse:
            raise ValueError("fused halo path needs a uniform fully-covered box layout")
        self.fused = can_fuse if fused is None else fused
        if exchange not in ("nccl", "peer"):
            raise ValueError(f"exchange must be 'nccl' or 'peer', not {exchange!r}")
        self.exchange = exchange if (self.fused and world > 1) else "nccl"
        if self.exchange == "peer":
            # faces on other ranks read over NVLink by the march itself (peer.py); ranks that
            # share a GPU are ordered by the host instead of the device barrier
            from .peer import PeerFused, ranks_share_device

            shared = ranks_share_device(mf.device)
            self.fh = PeerFused.connect(self.a, self.b, geom, barrier="host" if shared else "device",
                                        max_rows=march_rows)
            if shared:
                self.use_graph = False
        else:
            self.fh = march.FusedHalo(self.a, self.b, geom, march_rows, fill_plan=self.plan) if self.fused else None
        self._graph = None
        self._long = None  # one-rank: LONG_PAIRS captured pairs per replay (see advance)
        self._graph_pairs = 2 if (not self.fused and world == 1) else 1
        self._primed = False
        self.steps_done = 0

    @property
    def current(self) -> MultiFab:
        return self.a if self.steps_done % 2 == 0 else self.b

    @property
    def launches_per_step(self) -> int:
        if self.fused:
            # multi-rank: march (boundary and interior columns as two launches when both
            # exist), pack, unpack (+ x-halo refresh when an x face is remote)
            if self.exchange == "peer":
                return 1 + (self.fh.barrier is not None)  # march + device barrier
            if self.fh.remote:
                return 3 + (self.fh._remote_x is not None) + (self.fh.comm is not None)
            return 1
        # multi-rank: pack, local copies, interior sweep, unpack, boundary sweep
        return 5 if self.a.dm.nranks > 1 else 2

    def reset(self) -> None:
        """Call after modifying ``a`` from outside: restart at step 0."""
        self.steps_done = 0
        self._primed = False

    def close(self) -> None:
        """Release the captured graph.  Multi-rank: call before
        ``destroy_process_group`` -- a live graph holding NCCL work blocks the
        communicator's teardown."""
        import torch

        if self._graph is not None:
            torch.cuda.synchronize()
            self._graph = None
            self._long = None

    def _step(self, old: MultiFab, new: MultiFab) -> None:
        if self.fused:  # b -> a steps walk backwards: they start where a -> b ended (L2)
            self.fh.step(new, old, self.params, reverse=old is self.b)
        elif old.dm.nranks > 1:  # halo messages overlap the interior sweep
            overlapped_step(new, old, self.geom, self.params, self.plan, self.schedule, self.zmerge)
        else:
            fill_boundary(old, self.geom, self.plan)
            heat_step(new, old, self.geom, self.params, self.schedule, zmerge=self.zmerge)

    def _capture(self):
        import torch

        from .multifab import snapshots_in_capture

        # warm the plans (device tables, tensor maps) outside capture
        self._step(self.a, self.b)
        self._step(self.b, self.a)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), snapshots_in_capture():
            with torch.cuda.graph(g, stream=s):
                # the reference loop's fast path alternates each field's packed-halo buffers
                # once per pair of steps: the unfused one-rank graph holds two pairs, so its
                # frozen pointers repeat exactly with every replay
                for _ in range(self._graph_pairs):
                    self._step(self.a, self.b)
                    self._step(self.b, self.a)
        torch.cuda.current_stream().wait_stream(s)
        self._graph = g
        if self._check_graph:
            self._verify_capture()
        elif self.LONG_PAIRS > 1:
            # one rank: a second graph chaining LONG_PAIRS captured pairs; each replay of the
            # pair graph costs a graph launch (~1.4 us per C2 step at 2 steps per replay)
            gl = torch.cuda.CUDAGraph()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s), snapshots_in_capture():
                with torch.cuda.graph(gl, stream=s):
                    for _ in range(self.LONG_PAIRS * self._graph_pairs):
                        self._step(self.a, self.b)
                        self._step(self.b, self.a)
            torch.cuda.current_stream().wait_stream(s)
            self._long = gl

    def _verify_capture(self) -> None:
        """Multi-rank: replay the captured pair once and redo the same two
        steps eagerly from the same state; keep the graph only if every rank
        got identical bytes.  Leaves the state two steps ahead (eager)."""
        import torch
        import torch.distributed as dist

        a = self.a
        saved = [a.data.clone()]
        if self.fused:
            saved.append(self.fh.xh[id(a)].clone())
        self._graph.replay()
        got = a.data.clone()
        a.data.copy_(saved[0])
        if self.fused:
            self.fh.xh[id(a)].copy_(saved[1])
        self._step(self.a, self.b)
        self._step(self.b, self.a)
        same = torch.equal(got.view(torch.int64), a.data.view(torch.int64))
        flag = torch.tensor([1 if same else 0], dtype=torch.int32, device=a.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) != 1:
            self._graph = None
            self.use_graph = False

    def advance(self, n: int, finalize: bool = True) -> MultiFab:
        """Advance ``n`` steps; returns the MultiFab holding the state (all
        ghosts filled when ``finalize``)."""
        if self.fused and not self._primed:
            self.fh.prime(self.current, self.plan)
            self._primed = True
        k = 0
        if self.use_graph:
            if self.steps_done % 2 and n - k >= 3:  # realign to the captured a -> b -> a pair
                self._step(self.b, self.a)
                self.steps_done += 1
                k += 1
            # capturing runs two real steps, four when the capture is verified
            need = 4 if self._check_graph else 2
            if self.steps_done % 2 == 0 and self._graph is None and n - k >= need:
                self._capture()
                self.steps_done += need
                k += need
            if self.steps_done % 2 == 0 and self._long is not None:
                while n - k >= 2 * self._graph_pairs * self.LONG_PAIRS:
                    self._long.replay()
                    self.steps_done += 2 * self._graph_pairs * self.LONG_PAIRS
                    k += 2 * self._graph_pairs * self.LONG_PAIRS
            if self.steps_done % 2 == 0 and self._graph is not None:
                while n - k >= 2 * self._graph_pairs:
                    self._graph.replay()
                    self.steps_done += 2 * self._graph_pairs
                    k += 2 * self._graph_pairs
        while k < n:
            old, new = (self.a, self.b) if self.steps_done % 2 == 0 else (self.b, self.a)
            self._step(old, new)
            self.steps_done += 1
            k += 1
        if finalize:
            self.finalize()
        return self.current

    def finalize(self) -> None:
        """Refresh every ghost of the current state (one FillBoundary; only the
        fused path leaves edge/corner ghosts stale between steps)."""
        if self.fused:
            fill_boundary(self.current, self.geom, self.plan)


def _nccl_world() -> bool:
    """Multi-rank steps may be graph-captured: NCCL collectives are."""
    if os.environ.get("TM_MULTI_GRAPH", "1") == "0":
        return False
    try:
        import torch.distributed as dist

        return dist.is_initialized() and dist.get_backend() == "nccl"
    except (ImportError, RuntimeError):  # pragma: no cover
        return False
