"""Benchmark: fp64 cell-updates/s of steps x (FillBoundary + heat sweep).

Workload: BASELINE.json config 2 (C2) -- periodic 256^3, max_grid_size 64
(64 boxes of 64^3), 1 ghost, 1 component, tile (1024,8,8), seeded
Gaussian-plus-noise init, D=1, dt = 0.9*dx^2/6.  A "step" is one
FillBoundary plus one heat sweep over every box.  Boxes are distributed
over the ranks by DistributionMapping (strong scaling: total work fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank drives one GPU; the timed region is bracketed by a
barrier + cuda synchronize, timed with CUDA events on the launching stream,
and the max over ranks is reported.  Rank 0 prints one JSON line.

``--impl reference`` times the reference's CPU path (restated in C,
oracle/tm_oracle.c: tag copies + the four-loop tiled heat kernel, OpenMP
over all host cores) on rank 0 on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 cell-updates/sec (stencil sweep incl. FillBoundary) and % of HBM roofline"
UNIT = "cell-updates/s"
BYTES_PER_CELL = 16  # algorithmic: read u_old + write u_new


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the config's domain split over the GPUs; weak: a slab of the config's "
                         "per-GPU share at 8 GPUs per rank (Workload.weak)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--zmerge", action="store_true", help="fuse z-stacked tiles into one CTA k-march")
    ap.add_argument("--unfused", action="store_true",
                    help="reference step structure (FillBoundary kernel + tiled sweep) instead of the fused step")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true", help="skip the two-jobs-in-flight e2e variant")
    ap.add_argument("--configs", default="C3,C4,C5",
                    help="other BASELINE configs measured after the headline at N=1 ('' to skip)")
    ap.add_argument("--exchange", choices=["auto", "nccl", "peer"], default="auto",
                    help="multi-GPU halos: NCCL messages, or peer: the march reads other ranks' faces over "
                         "NVLink (auto: peer when every rank can map its peers and a short run matches NCCL)")
    ap.add_argument("--hot-steps", type=int, default=2000,
                    help="untimed steps run right before the timed region (keeps clocks up)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic(config_name: str, fused: bool = False):
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as fh:
            d = json.load(fh)
        key = "fused_step" if fused else "heat_sweep"
        return d.get(key, {}).get(config_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU arm: the reference path restated in C (oracle), rank 0 only
# ---------------------------------------------------------------------------
def cpu_reference_rate(w, budget_s: float, steps: int | None = None, boxes: int | None = None,
                       threads: int | None = None):
    """(rate, cores, sample description, steps run, boxes used) for the
    reference CPU path (tag fill + four-loop tiled heat; all host threads, or
    ``threads``) on the first ``boxes`` boxes of the workload."""
    import numpy as np

    from oracle import oracle as orc
    from paper_1604_03570_b200 import BoxArray, Geometry, HeatParams, make_init
    from paper_1604_03570_b200.box import decompose
    from paper_1604_03570_b200.fillplan import build_fill_plan_units

    # every host core this process may run on (torchrun exports OMP_NUM_THREADS=1; num_threads(n)
    # in tm_oracle.c overrides it)
    threads = len(os.sched_getaffinity(0)) if threads is None else threads
    ba = BoxArray.chop(w.domain, w.max_grid_size)
    valids = list(ba)
    geom = Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    plan = build_fill_plan_units(valids, geom, w.nghost, grids=valids)
    glob = make_init(w)
    old = orc.HostMF(valids, w.ncomp, w.nghost)
    old.from_global(glob)
    new = orc.HostMF(valids, w.ncomp, w.nghost)
    c = HeatParams.stable(1.0, geom.dx).coefficients()
    nb = len(valids) if boxes is None else max(1, min(len(valids), boxes))
    tags = orc.tags_array([t for t in plan.tags if t.dst_unit < nb])
    tiles = orc.tiles_array([(u, t) for u in range(nb) for t in decompose(valids[u], w.tile_size)])
    cells = sum(v.ncells for v in valids[:nb]) * w.ncomp
    # warm-up pass (page-in, thread pool)
    orc.fill_boundary(old, tags, threads)
    orc.heat_step(new, old, tiles, c[:3], c[3], threads)
    n = 0
    t0 = time.perf_counter()
    while True:
        orc.fill_boundary(old, tags, threads)
        orc.heat_step(new, old, tiles, c[:3], c[3], threads)
        old, new = new, old
        n += 1
        el = time.perf_counter() - t0
        if (steps is not None and n >= steps) or (steps is None and el >= budget_s):
            break
    rate = cells * n / el
    sample = (f"{w.name}: {nb} of {len(valids)} boxes ({cells} cells), {n} x (tag FillBoundary + tiled 4-loop heat), "
              f"oracle/tm_oracle.c OpenMP x{threads}, {el:.2f} s")
    return rate, threads, sample, n, nb, el


REF_INSTALL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")


def numba_reference_rate(w, threads: int, steps: int | None, budget_s: float, warmup: int = 1):
    """The UNMODIFIED reference (pip-installed into baseline/_ref by __graft_entry__.build())
    through its own public API and timing loop shape (tilemesh/bench.py:183-206: fill_boundary
    + heat_step per step, JIT warmed outside the timed region) on workload ``w`` with all
    boxes.  Returns None when the install or numba is absent on this host.  ``steps`` is
    capped so the timed loop stays within ``budget_s`` seconds."""
    if not os.path.isdir(os.path.join(REF_INSTALL, "tilemesh")):
        return None
    sys.path.insert(0, REF_INSTALL)
    try:
        from tilemesh.bench import RunConfig, _setup, _steppers
        from tilemesh.level import build_fill_plan, fill_boundary
    except Exception:  # numba / matplotlib missing on this host
        return None
    finally:
        sys.path.remove(REF_INSTALL)
    if w.ncomp != 1 or w.nghost != 1:
        return None  # the reference's bench set-up is one component, one ghost layer
    e = w.domain.extents
    cfg = RunConfig(nx=e[0], ny=e[1], nz=e[2], max_grid_size=w.max_grid_size, tile_size=tuple(w.tile_size),
                    threads=threads, steps=0)
    geom, old = _setup(cfg)  # the reference's own cosine init: values change no code path
    new = old.clone_empty()
    plan = build_fill_plan(old, geom)
    step, _ = _steppers(cfg, geom, old)
    t0 = time.perf_counter()
    for _ in range(max(1, warmup)):  # JIT + page-in
        fill_boundary(old, geom, plan, threads)
        step(old, new)
        old, new = new, old
    t0 = time.perf_counter()
    fill_boundary(old, geom, plan, threads)
    step(old, new)
    old, new = new, old
    per = time.perf_counter() - t0
    cap = max(1, int(budget_s / max(per, 1e-9)))
    n = cap if steps is None else max(1, min(steps, cap))
    t0 = time.perf_counter()
    for _ in range(n):
        fill_boundary(old, geom, plan, threads)
        step(old, new)
        old, new = new, old
    el = time.perf_counter() - t0
    rate = w.cells * n / el
    sample = (f"{w.name}: all {len(old.units)} boxes, {n} x (fill_boundary + heat_step) of the unmodified reference "
              f"(tilemesh 0.1.0, numba, baseline/_ref), threads={threads}, {el:.2f} s")
    return rate, threads, sample, n, el


def run_reference(args, w):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_1604_03570_b200 as tm

    nboxes = len(tm.BoxArray.chop(w.domain, w.max_grid_size))
    # bound each step: size the per-step sample so the whole run is ~a minute
    total = max(args.steps + args.warmup, 1)
    per_step_budget = 60.0 / total
    probe_rate, _, _, _, _, _ = cpu_reference_rate(w, budget_s=1.0, steps=1, boxes=1)
    box_cells = w.cells // nboxes
    boxes = max(1, int(per_step_budget * probe_rate / box_cells))
    if args.warmup:
        cpu_reference_rate(w, 0, steps=args.warmup, boxes=boxes)
    rate, cores, sample, n, nb, el = cpu_reference_rate(w, 0, steps=args.steps, boxes=boxes)
    port = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
            "ms_per_step": el / n * 1e3, "sample_boxes_per_step": nb}
    # the unmodified reference itself, when its install travelled to this host (all boxes per
    # step; steps capped to ~60 s of timed work)
    threads = len(os.sched_getaffinity(0))
    ref = None
    try:
        ref = numba_reference_rate(w, threads, args.steps, 60.0, warmup=max(1, min(args.warmup, 3)))
    except Exception as exc:  # never lose the arm to the optional leg
        port["reference_error"] = f"{type(exc).__name__}: {exc}"[:200]
    if ref is not None:
        r_rate, r_cores, r_sample, r_n, r_el = ref
        value, ms, cpu = r_rate, r_el / r_n * 1e3, {"value": r_rate, "unit": UNIT, "cores": r_cores,
                                                    "kind": "reference", "sample": r_sample, "steps_timed": r_n,
                                                    "port": port}
    else:
        value, ms, cpu = rate, el / n * 1e3, port
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{w.name}: periodic {w.domain.extents[0]}x{w.domain.extents[1]}x"
                               f"{w.domain.extents[2]}, max_grid_size {w.max_grid_size} "
                               f"({nboxes} boxes), nghost {w.nghost}, ncomp {w.ncomp}, tile {w.tile_size}",
                   "sample_boxes_per_step": nboxes if ref is not None else nb},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def local_slab(mf):
    """Bounding box of this rank's boxes and whether it is exactly their union
    (always so for the slab DistributionMapping of the BASELINE configs):
    host transfers then move the rank's own slab only."""
    from paper_1604_03570_b200.box import bounding_box

    boxes = [mf.units[u].valid for u in mf.local_units]
    bb = bounding_box(boxes)
    return bb, bb.ncells == sum(b.ncells for b in boxes)


def host_init(args, w, slab, rank):
    """Pinned host array (ncomp, nz, ny, nx) of this rank's slab initial data.
    Strong scaling: the config's seeded global init, sliced;
    weak scaling: seeded uniform values per rank (no rank builds the global)."""
    import numpy as np
    import torch

    import paper_1604_03570_b200 as tm

    e = slab.extents
    if args.scaling == "weak":
        rng = np.random.default_rng(1000 + rank)
        arr = rng.random((w.ncomp, e[2], e[1], e[0]))
    else:
        glob = tm.make_init(w)
        sl = tuple(slice(slab.lo[d], slab.hi[d] + 1) for d in (2, 1, 0))
        arr = np.ascontiguousarray(glob[(slice(None),) + sl])
        del glob
    return torch.from_numpy(arr).pin_memory()


def run_ours(args, w):
    import torch
    import torch.distributed as dist

    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200 import halo
    from paper_1604_03570_b200.runner import HeatRunner

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE is {world}")
    # one process per GPU; TM_DIST_BACKEND=gloo lets several ranks share one GPU to
    # smoke-test the multi-rank path (host-staged halos) -- never used for numbers
    backend = os.environ.get("TM_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    if args.scaling == "weak":
        w = w.weak(world)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    mf = tm.MultiFab(ba, w.ncomp, w.nghost)
    slab, exact = local_slab(mf)
    if not exact:
        raise SystemExit("bench.py: this rank's boxes do not form a slab")
    host_in = host_init(args, w, slab, rank)
    mf.from_global(host_in.to(dev), domain=slab)
    params = tm.HeatParams.stable(1.0, geom.dx)
    plan = tm.build_fill_plan(mf, geom)
    sched = tm.build_schedule(mf, w.tile_size)
    runner, peer_check = make_runner(args, HeatRunner, mf, geom, params, sched, plan, world, dev)
    local_cells = sum(ba[u].ncells for u in mf.local_units) * w.ncomp
    total_cells = w.cells * w.ncomp

    # --- warm-up (includes graph capture) --------------------------------
    runner.advance(max(args.warmup, 3))
    barrier()

    # --- timed region: K steps, CUDA events on the launching stream -----
    # Two hygiene steps around it: (1) the clock sampler's start-up pause would leave the GPU
    # idle for ~0.15 s right before the timed region (clocks drop; the first ~20 steps then ran
    # ~10 % slow), so untimed steps keep it busy until the barrier; (2) a short device sleep
    # queued before ev0 lets the host enqueue the K steps' graph replays behind it, so no host
    # issue gap is inside the timed region.  ev_mid splits the K steps (graph replays) from the
    # closing FillBoundary, so the step kernel's launch time is measured directly.
    stream = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev_mid = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        runner.advance(args.hot_steps + (args.hot_steps % 2), finalize=False)
        barrier()
        torch.cuda._sleep(400_000)  # ~0.2 ms at 1.965 GHz
        ev0.record(stream)
        runner.advance(args.steps, finalize=False)
        ev_mid.record(stream)
        runner.finalize()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    steps_ms = ev0.elapsed_time(ev_mid)
    t = torch.tensor([ms, steps_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, steps_ms_max = (float(v) for v in t.tolist())
    value = total_cells * args.steps / (ms_max * 1e-3)

    # --- per-launch kernel times (eager, CUDA events on the launching stream) --
    # The GPU queue stays ahead of the Python issue loop (each launch is tens of
    # microseconds of device time), so event deltas are device time.
    def timed(fn, nrep=40):
        cur = runner.current
        other = runner.b if cur is runner.a else runner.a
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(nrep + 1)]
        for _ in range(3):
            fn(cur, other)
            cur, other = other, cur
        barrier()
        evs[0].record(stream)
        for r in range(nrep):
            fn(cur, other)
            cur, other = other, cur
            evs[r + 1].record(stream)
        barrier()
        return sum(evs[r].elapsed_time(evs[r + 1]) for r in range(nrep)) / nrep

    if runner.fused:
        def fused_step(o, n):
            runner.fh.step(n, o, params)
        runner.fh.prime(runner.current, plan)
        kern_ms = timed(fused_step)
        kern_name = ("march_kernel<PACKED,SCATTER,NBRH> (tm_heat_march TM_HALO_FUSED_NBR: sweep + fused "
                     "face-halo exchange)")
        if world > 1 and runner.exchange == "peer":
            kern_name += (" with remote faces TMA-loaded from the peers' storage over NVLink (tm_heat_march_peer)"
                          " + tm_peer_barrier")
        elif world > 1:
            kern_name += " + NCCL halo exchange of remote faces"
    fill_ms = timed(lambda o, n: tm.fill_boundary(o, geom, plan))
    sweep_ms = timed(lambda o, n: tm.heat_step(n, o, geom, params, sched, zmerge=args.zmerge))
    if not runner.fused:
        kern_ms = sweep_ms
        kern_name = "heat_step sweep (column march when eligible, else tile kernel)"
    eager_ms = kern_ms
    if runner.fused and runner.use_graph:
        # ev0 -> ev_mid in the timed region is exactly K step launches (graph replays)
        kern_ms = steps_ms / args.steps
    runner.reset()  # state was advanced outside the runner's bookkeeping
    peak, peak_src = peaks()

    # --- the reference-shaped loop: fill_boundary(old); heat_step(new, old) ---
    # (a) captured as a CUDA graph of step pairs (HeatRunner fused=False); (b) issued eagerly from a
    # Python loop exactly as a drop-in caller writes it.  Both on the packed-x-halo fast path once
    # the first heat_step has run.
    refloop = None
    if world == 1:
        ref_mf = mf.clone_empty()
        ref_mf.data.copy_(runner.current.data)
        rr = HeatRunner(ref_mf, geom, params, sched, plan, fused=False)
        rr.advance(4)
        torch.cuda.synchronize()
        torch.cuda._sleep(400_000)
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        rr.advance(args.steps)
        r1.record(stream)
        torch.cuda.synchronize()
        graph_ms = r0.elapsed_time(r1) / args.steps
        old_, new_ = rr.current, (rr.b if rr.current is rr.a else rr.a)
        for _ in range(4):
            tm.fill_boundary(old_, geom, plan)
            tm.heat_step(new_, old_, geom, params, sched)
            old_, new_ = new_, old_
        torch.cuda.synchronize()
        r0.record(stream)
        for _ in range(args.steps):
            tm.fill_boundary(old_, geom, plan)
            tm.heat_step(new_, old_, geom, params, sched)
            old_, new_ = new_, old_
        r1.record(stream)
        torch.cuda.synchronize()
        eager_ms = r0.elapsed_time(r1) / args.steps
        fast = bool(old_.xh_current() and old_.ghosts_current() is False)
        refloop = {"graph": {"ms_per_step": graph_ms, "value": total_cells / (graph_ms * 1e-3),
                             "roofline_frac": BYTES_PER_CELL * local_cells / (graph_ms * 1e-3) / 1e9 / peak},
                   "eager_python": {"ms_per_step": eager_ms, "value": total_cells / (eager_ms * 1e-3),
                                    "roofline_frac": BYTES_PER_CELL * local_cells / (eager_ms * 1e-3) / 1e9 / peak},
                   "packed_x_halo_path": fast,
                   "how": "fill_boundary(old, geom, plan); heat_step(new, old, geom, params, sched) per step, "
                          "K steps between CUDA events; (graph) HeatRunner(fused=False) replaying captured pairs"}
        rr.close()
        del rr, ref_mf
    achieved = BYTES_PER_CELL * local_cells / (kern_ms * 1e-3) / 1e9
    ghost_cells = sum(t.dst_box.ncells for t in plan.tags if mf.unit_owner[t.dst_unit] == mf.rank) * w.ncomp
    fill_gbs = 16 * ghost_cells / (fill_ms * 1e-3) / 1e9

    # --- end-to-end through the public API with host buffers -------------
    # one job = upload this rank's slab of phi0 from pinned host memory, run the
    # config's steps (graph replays), read back the final slab and the checksum.
    job_steps = w.steps
    host_out = torch.empty_like(host_in).pin_memory()
    e2e_runs = 3
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    side = torch.cuda.Stream(dev)
    for it in range(e2e_runs + 1):  # run 0 is an untimed warm-up (allocator, side stream)
        if it == 1:
            barrier()
            e0.record(stream)
        g = host_in.to(dev, non_blocking=True)
        runner.a.from_global(g, domain=slab)
        runner.reset()
        out = runner.advance(job_steps)
        # the checksum (a latency-bound serial chain per box, bit-exact with the
        # reference) runs on a side stream while phi is gathered and read back
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            csum = out.reduce_sum_device()
        host_out.copy_(out.to_global(domain=slab))
        stream.wait_stream(side)
        host_csum = float(csum.item())
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / e2e_runs
    te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    e2e_value = total_cells * job_steps / (e2e_ms * 1e-3)
    h2d = host_in.numel() * 8 * world  # every rank uploads its own slab (slabs tile the domain)
    d2h = (host_out.numel() * 8 + 8) * world

    # --- e2e, job stream: two jobs in flight on two CUDA streams ----------
    pipe = None
    # one GPU only: concurrent graphs on two streams must not interleave one NCCL communicator
    if not args.no_pipeline and world == 1:
        pipe = pipelined_e2e(runner, HeatRunner, mf, geom, params, sched, plan, args, host_in, slab, job_steps,
                             host_csum, total_cells, barrier, dev, stream)
        runner.reset()

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            rate, cores, sample, _, _, _ = cpu_reference_rate(w, args.cpu_seconds)
            rate1, _, sample1, _, _, _ = cpu_reference_rate(w, args.cpu_seconds / 2, threads=1)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                   "one_core": {"value": rate1, "cores": 1, "sample": sample1}}
            try:  # the unmodified reference beside the port, when its install is on this host
                ref = numba_reference_rate(w, cores, None, args.cpu_seconds)
                if ref is not None:
                    cpu["unmodified_reference"] = {"value": ref[0], "unit": UNIT, "cores": ref[1],
                                                   "kind": "reference", "sample": ref[2]}
            except Exception as exc:
                cpu["unmodified_reference"] = {"error": f"{type(exc).__name__}: {exc}"[:200]}
        traffic = profile_traffic(w.name, runner.fused)
        others = config_records(args, peak) if world == 1 and args.configs else None
        launches_per_step = runner.launches_per_step
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic" + (" (seeded uniform per rank)" if args.scaling == "weak" else
                                   " (seeded init of BASELINE.json's config)"),
            "config": {
                "workload": f"{w.name}: periodic {w.domain.extents[0]}x{w.domain.extents[1]}x{w.domain.extents[2]}, "
                            f"max_grid_size {w.max_grid_size} ({len(ba)} boxes), nghost {w.nghost}, "
                            f"ncomp {w.ncomp}, tile {w.tile_size}",
                "step": "FillBoundary + heat sweep over all boxes",
                "l2": f"inputs larger than L2: {2 * local_cells * 8 / 1e6:.0f} MB streamed per step per GPU "
                      f"vs 126 MB L2",
                "parallelism": f"dm{world} (contiguous box slabs, one process per GPU, " + (
                    "peer halos: faces read over NVLink inside the march, one device barrier per step)"
                    if runner.exchange == "peer" else "NCCL halo exchange)"),
                "exchange": runner.exchange, "peer_check": peer_check,
                "cuda_graph": runner.use_graph, "zmerge": args.zmerge,
                "step_impl": ("fused: one persistent column-march launch per step; y/z halos read from the face "
                              "neighbours' valid cells, x halos from packed buffers the previous step's epilogue "
                              "wrote (FillBoundary fused); edges/corners refreshed by one FillBoundary per "
                              "advance()" if runner.fused else
                              "FillBoundary kernel + tiled heat sweep (2 launches per step)"),
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "traffic_note": "ncu dram__bytes_read+write of one cold launch (profiles/ncu_summary.json, static); "
                                "write-back of the last ~40 MB lands after the kernel ends",
                "kernel": kern_name,
                "bytes_per_launch": BYTES_PER_CELL * local_cells, "avg_launch_ms": kern_ms,
                "avg_launch_ms_how": "timed region ev0->ev_mid (K graph-replayed step launches) / K"
                if runner.fused and runner.use_graph else "eager launches between CUDA events",
                "eager_launch_ms": eager_ms,
                "peak_source": peak_src,
                # north_star quotes "roughly 8 TB/s"; SURVEY.md §8d asks for both figures
                "frac_vs_nominal_8000_gbs": achieved / 8000.0,
                # context, static: what a plain copy of one C2 launch's bytes does at this size
                **({"same_size_copy_note":
                     "a plain copy of 134 MB read + 134 MB written in one launch (296 CTAs) takes ~46.1 us with "
                     "equal static shares (0.89 of the peak) and 43.4 us with dynamic shares (0.94): "
                     "tools/micro/sm_rate.cu, profiles/r02/sm_rate_copy_probe.txt"}
                   if w.name == "C2" and world == 1 else {}),
            },
            "unfused_components": {"fill_boundary_ms": fill_ms, "fill_ghost_gbs": fill_gbs,
                                   "ghost_cells": ghost_cells, "heat_step_ms": sweep_ms,
                                   "note": "each op timed alone in a loop of itself (no packed-halo hand-over)"},
            "reference_loop": refloop,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / job_steps,
                    "d2h_bytes_per_step": d2h / job_steps,
                    "job": f"each rank uploads its slab of phi0 (pinned) + {job_steps} steps + downloads its slab "
                           f"+ checksum",
                    "ms_per_job": e2e_ms, "checksum": host_csum, "pipelined": pipe},
            "gpu_launches": launches_per_step * args.steps + (1 if runner.fused else 0),
            "clocks": clocks.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if others is not None:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    runner.close()  # before the process group goes: a live graph may hold NCCL work
    halo.close_comm()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def make_runner(args, HeatRunner, mf, geom, params, sched, plan, world, dev):
    """The bench runner.  Multi-GPU with ``--exchange auto|peer``: the peer path (peer.py) when
    every rank can map its peers' memory; under ``auto`` it is kept only if 4 steps of it give
    the same bytes as 4 steps of the NCCL path from the same state on every rank."""
    import torch
    import torch.distributed as dist

    kw = dict(use_graph=not args.no_graph, zmerge=args.zmerge, fused=False if args.unfused else None)
    if world == 1 or args.unfused or args.exchange == "nccl":
        return HeatRunner(mf, geom, params, sched, plan, **kw), None
    from paper_1604_03570_b200.peer import peer_face_table

    ok = 1
    why = "ok"
    try:
        peer_face_table(mf, geom)
        n = torch.cuda.device_count()
        if os.environ.get("TM_DIST_BACKEND", "nccl") == "nccl" and n < world:
            ok, why = 0, f"{n} visible GPUs < {world} ranks: peers' memory cannot be mapped"
        elif not all(torch.cuda.can_device_access_peer(dev.index, j) for j in range(n) if j != dev.index):
            ok, why = 0, "no peer access between the GPUs"
    except ValueError as e:
        ok, why = 0, str(e)
    flag = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) != 1:
        if args.exchange == "peer":
            raise SystemExit(f"bench.py: --exchange peer not possible: {why}")
        return HeatRunner(mf, geom, params, sched, plan, **kw), {"used": False, "why": why}
    if args.exchange == "peer":
        return HeatRunner(mf, geom, params, sched, plan, exchange="peer", **kw), {"used": True, "checked": False}
    # auto: same 4 steps through both paths (copies of the initial state), bytes compared on every rank
    ref_mf = mf.clone_empty()
    ref_mf.data.copy_(mf.data)
    ref = HeatRunner(ref_mf, geom, params, sched, plan, use_graph=False)
    want = ref.advance(4).data.clone()
    ref.close()
    del ref, ref_mf
    probe_mf = mf.clone_empty()
    probe_mf.data.copy_(mf.data)
    try:  # IPC mapping can fail (e.g. a device not visible); every collective of the setup is done by then
        probe = HeatRunner(probe_mf, geom, params, sched, plan, exchange="peer", use_graph=False)
        ok, why = 1, "ok"
    except Exception as e:  # noqa: BLE001 -- any setup failure means: use NCCL
        probe, ok, why = None, 0, f"peer setup failed: {e}"[:200]
    flag = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) != 1:
        if probe is not None:
            probe.fh.close()
        return HeatRunner(mf, geom, params, sched, plan, **kw), {"used": False, "why": why}
    same = torch.equal(probe.advance(4).data.view(torch.int64), want.view(torch.int64))
    if probe.fh.barrier is not None and probe.fh.barrier.timed_out():
        same = False
    torch.cuda.synchronize()
    dist.barrier()
    probe.fh.close()
    del probe, probe_mf, want
    flag = torch.tensor([1 if same else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) != 1:
        return HeatRunner(mf, geom, params, sched, plan, **kw), {"used": False, "why": "4-step check vs NCCL differed"}
    runner = HeatRunner(mf, geom, params, sched, plan, exchange="peer", **kw)
    return runner, {"used": True, "checked": "4 steps bit-identical to the NCCL path on every rank"}


def pipelined_e2e(runner, HeatRunner, mf, geom, params, sched, plan, args, host_in, slab, job_steps, host_csum,
                  total_cells, barrier, dev, stream):
    """The e2e job stream with two jobs in flight: each job as in ``e2e``
    (pinned upload, steps, gather + pinned download, checksum), alternating
    between two runners / CUDA streams so one job's PCIe copies overlap the
    other's steps; host reads after the last job."""
    import torch

    runner2 = HeatRunner(mf.clone_empty(), geom, params, sched, plan, use_graph=runner.use_graph,
                         zmerge=args.zmerge, fused=runner.fused)
    runners = [runner, runner2]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    dev_in = [torch.empty_like(host_in, device=dev) for _ in range(2)]
    dev_out = [torch.zeros_like(host_in, device=dev) for _ in range(2)]
    host_outs = [torch.empty_like(host_in).pin_memory() for _ in range(2)]
    pipe_jobs = 8
    csums = []
    sides = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]

    def job(j):
        r, st, sd = runners[j % 2], streams[j % 2], sides[j % 2]
        with torch.cuda.stream(st):
            st.wait_stream(sd)  # job j-2's checksum has read the field
            dev_in[j % 2].copy_(host_in, non_blocking=True)
            r.a.from_global(dev_in[j % 2], domain=slab)
            r.reset()
            o = r.advance(job_steps)
            o.to_global(domain=slab, out=dev_out[j % 2])
            sd.wait_stream(st)
            with torch.cuda.stream(sd):  # checksum beside the download
                csums.append(o.reduce_sum_device().clone())  # the scratch total is reused
            host_outs[j % 2].copy_(dev_out[j % 2], non_blocking=True)

    for j in range(2):  # untimed: captures runner2's graph, warms both streams
        job(j)
    barrier()
    csums.clear()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for st in streams + sides:
        st.wait_stream(stream)
    for j in range(pipe_jobs):  # job j reuses job j-2's buffers on the same stream (ordered)
        job(j)
    for st in streams + sides:
        stream.wait_stream(st)
    p1.record(stream)
    barrier()
    pipe_ms = p0.elapsed_time(p1) / pipe_jobs
    pipe_ok = all(float(c.item()) == host_csum for c in csums) and torch.equal(host_outs[0], host_outs[1])
    runner2.close()
    return {"value": total_cells * job_steps / (pipe_ms * 1e-3), "unit": UNIT, "jobs": pipe_jobs,
            "in_flight": 2, "ms_per_job": pipe_ms, "checksums_match_serial": bool(pipe_ok),
            "how": "same job as e2e; jobs alternate over two runners / CUDA streams so uploads and "
                   "downloads overlap the other job's steps"}


def config_records(args, peak):
    """BASELINE.json's other configs on this GPU (N=1), so their rates are in the
    driver's record and not only in the builder's logs: C3 and C5 heat (fused,
    chained steps, graph-replayed; device-side uniform init -- the values change no
    code path) and C4 (GSRB solve, colour-split).  Each: cell-updates/s over K steps
    timed with CUDA events (inputs larger than L2), and the fraction of the HBM peak
    on the algorithmic bytes (16 B per heat update, 24 B per GSRB update).  A config
    that fails reports its error instead of a number."""
    import torch

    import paper_1604_03570_b200 as tm
    from paper_1604_03570_b200.runner import HeatRunner

    out = {}

    def timed(fn, reps):
        torch.cuda.synchronize()
        torch.cuda._sleep(400_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(reps)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for name in args.configs.split(","):
        name = name.strip()
        if not name:
            continue
        w = tm.CONFIGS[name]
        try:
            geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
            ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
            cells = w.cells * w.ncomp
            if w.kernel == "heat":
                mf = tm.MultiFab(ba, w.ncomp, w.nghost, zero=False)
                mf.data.uniform_()
                r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), w.tile_size)
                k = max(4, min(w.steps, 20))
                r.advance(k)  # warm-up: plans, graph capture
                ms = timed(lambda n: r.advance(n, finalize=False), k)
                rec = {"value": cells / (ms * 1e-3), "ms_per_step": ms, "steps": k,
                       "roofline_frac": 16 * cells / (ms * 1e-3) / 1e9 / peak, "bytes_per_update": 16,
                       "step_impl": "fused" if r.fused else "unfused"}
                r.close()
                del r, mf
            else:
                phi = tm.MultiFab(ba, 1, 1)
                rhs = tm.MultiFab(ba, 1, 0)
                rhs.from_global(tm.make_init(w))
                tm.gsrb_solve(phi, rhs, geom, 2)  # warm-up
                ms = timed(lambda n: tm.gsrb_solve(phi, rhs, geom, n), w.steps)
                rec = {"value": cells / (ms * 1e-3), "ms_per_sweep": ms, "sweeps": w.steps,
                       "roofline_frac": 24 * cells / (ms * 1e-3) / 1e9 / peak, "bytes_per_update": 24,
                       "residual": tm.residual_maxnorm(phi, rhs, geom),
                       "note": "per sweep incl. the solve's split/merge and closing FillBoundary"}
                del phi, rhs
            rec["workload"] = (f"{name}: periodic {w.n}^3, max_grid_size {w.max_grid_size} ({len(ba)} boxes), "
                               f"nghost {w.nghost}, ncomp {w.ncomp}")
            rec["unit"] = UNIT
            out[name] = rec
        except Exception as e:  # noqa: BLE001 -- reported, the headline line still prints
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
        torch.cuda.empty_cache()
    # the 9-point 8th-order stencil ("wide4") on the C2 shape with the
    # 4 ghost layers it needs -- the fused runner (Kernel W2, neighbour-sourced halos, one
    # launch per step) and the reference loop (fill_boundary + wide4_step per step)
    try:
        import dataclasses

        w = dataclasses.replace(tm.CONFIGS["C2"], nghost=4)
        geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
        ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
        mf = tm.MultiFab(ba, 1, 4, zero=False)
        mf.data.uniform_()
        dt = tm.wide4_stable_dt(1.0, geom.dx)
        r = tm.Wide4Runner(mf, geom, 1.0, dt)
        k = 20
        r.advance(k)
        ms = timed(lambda n: r.advance(n, finalize=False), k)
        cells = w.cells
        old, new = r.a, r.b
        plan = tm.build_fill_plan(old, geom)

        def refloop(n):
            a_, b_ = old, new
            for _ in range(n):
                tm.fill_boundary(a_, geom, plan)
                tm.wide4_step(b_, a_, geom, 1.0, dt)
                a_, b_ = b_, a_

        refloop(2)
        ms_ref = timed(refloop, k)
        out["wide4_C2shape"] = {
            "value": cells / (ms * 1e-3), "ms_per_step": ms, "steps": k,
            "roofline_frac": 16 * cells / (ms * 1e-3) / 1e9 / peak, "bytes_per_update": 16,
            "step_impl": ("fused: one Kernel W2 launch per step, every 4-deep halo read from the face "
                          "neighbours' valid cells" if r.fused and r.nbr_halos else
                          "fused" if r.fused else "unfused"),
            "reference_loop": {"ms_per_step": ms_ref, "value": cells / (ms_ref * 1e-3),
                               "how": "fill_boundary (4 ghost layers) + wide4_step per step, eager: the fill is "
                                      "deferred and rides on the step's launch (tm_wide4_march_fill)"},
            "workload": f"wide4 (9-point 8th-order Laplacian, SURVEY §8f row 1): periodic {w.n}^3, "
                        f"max_grid_size {w.max_grid_size} ({len(ba)} boxes), nghost 4, ncomp 1",
            "unit": UNIT,
        }
        r.close()
        del r, mf
    except Exception as e:  # noqa: BLE001
        out["wide4_C2shape"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    torch.cuda.empty_cache()
    return out


def spawn_ranks(args) -> int:
    """``--gpus N`` outside torchrun: launch N single-GPU ranks of this script
    (torch.distributed.run, rendezvous on 127.0.0.1) and pass their output
    through; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    from paper_1604_03570_b200.configs import CONFIGS

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    w = CONFIGS[args.config]
    if args.impl == "reference":
        if args.scaling == "weak":
            w = w.weak(args.gpus)
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
