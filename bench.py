"""Benchmark: CCD queries/sec (FP64, delta=1e-6) on 1..8 B200, + FP64 roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3] [--queries Q] [--separation D]

Workload (default BASELINE config 3, the metric's "sharded across 1/2/4/8
GPUs" set): Q = 5e7 simulation-shaped queries (80% VF / 20% EE, delta=1e-6,
m_I=1e6, d=0, t_max=1), generated once from the index-addressable seeded
stream (paper_2009_13349_b200/workloads.py) and sliced contiguously across
the N ranks (strong scaling: rank r solves queries shard_bounds(Q, N, r),
identical data for every N).  `--config 1` etc. select the other BASELINE
sets at their BASELINE sizes.  One step = one batched solve of this rank's
shard.  Inputs (192 B per query) exceed the 126 MB L2 at every N, so no
flush is needed.

`--gpus N` without WORLD_SIZE in the environment re-launches this script
under torch.distributed.run with N ranks (one per GPU); the driver's own
torchrun launch is used as is.  No collective touches the data path: the
barrier and the max-over-ranks timing reduction are the only cross-rank
steps (results stay on each rank's GPU / host).

value  = device-timed throughput, inputs resident in HBM, CUDA events on the
         launching stream, barrier + synchronize on both sides, max over
         ranks: Q / max-rank time.
e2e    = the same through the public API (solve_batch) with pinned HOST
         inputs: every step copies the shard's points + kind host->device
         (on the API's copy stream, chunk by chunk under the solve) and reads
         back the compacted hit list (index, toi) with its count -- the
         reference consumer's result (ccdkit.scene keeps only hits,
         pkg/src/ccdkit/scene.py:321-326) -- by a copy-out kernel that moves
         only the live entries; all inside the timed region.
roofline = the dominant kernel of the step (by its CUDA-event time): its
         ALGORITHMIC FP64 flops per launch / its average duration.  Flops
         per check F_VF = 200, F_EE = 174 and per query P_VF = 248, P_EE =
         222; the check counts are the reference's own (the
         library counts, per stage, only checks on the reference's path:
         the lane tier counts the queries it finishes, the group tiers
         exclude speculative and re-run work).  peak = the DFMA rate measured
         on this box by libtccd_probe.so (FMA-counted; an FMA-free kernel is
         capped at 0.5 of it -- the rounding contract forbids DFMA).
cpu_baseline = the reference's own CPU path: ccdkit._kernel.solve_kernel
         (numba, from the git-ignored baseline/_ref install) over the same
         workload's queries in a spawn pool with one worker per host core,
         rank 0, every N, bounded sample; the C port of oracle/ stands in if
         the reference is not importable (kind "port").
--impl reference: that CPU path alone, same metric / config (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

F_CHECK = {0: 200, 1: 174}
P_QUERY = {0: 248, 1: 222}
METRIC = "CCD queries/sec (FP64, delta=1e-6) at 1/2/4/8 B200; % of FP64 roofline"
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
NAMES = {
    0: "config0: vertex-face, U[0,1]^3 + U[-0.5,0.5]^3 motion",
    1: "config1: 50% VF / 50% EE, half planted exact roots, half config-0 random",
    2: "config2: degenerate lattice families, delta in {1e-4,1e-6,1e-8}, m_I in {1e3,1e6}",
    3: "config3: simulation-shaped, 80% VF / 20% EE, edge 1e-2, offsets N(0,1e-3)/N(0,5e-3)",
    4: "config4: config-3 law (own seed stream), minimum separation d",
}
DEFAULT_Q = {0: 10_000, 1: 1_000_000, 2: 200_000, 3: 50_000_000, 4: 10_000_000}
KERNEL_NAMES = {"prologue": "prologue_kernel", "lane": "lane_kernel",
                "light": "engine_kernel (light tier)", "medium": "engine_kernel (medium tier)",
                "giant": "engine_kernel (giant tier)"}


def workload_desc(cfg: int, q: int, world: int, sep: float) -> dict:
    from paper_2009_13349_b200 import workloads as W
    return {"workload": NAMES[cfg], "baseline_config": cfg, "queries": q,
            "queries_per_gpu": q // world, "sharding": f"contiguous, {world} rank(s), one set",
            "delta": 1e-6 if cfg != 2 else "per-query", "max_checks": 1_000_000 if cfg != 2
            else "per-query", "separation": sep, "t_max": 1.0,
            "seed": f"PCG64(SeedSequence([{W.SEED_BASE}+{cfg}, block]))",
            "l2": "inputs > 126 MB L2 per step (no flush needed)" if q // world * 192 > 126e6
            else "inputs < L2: L2 flushed (256 MB write) before every timed step"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons while the timed region runs."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    for line in out.strip().splitlines():
                        self.rows.append([c.strip() for c in line.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peaks() -> dict:
    import ctypes
    so = os.path.join(ROOT, "paper_2009_13349_b200", "libtccd_probe.so")
    L = ctypes.CDLL(so)
    L.tccd_probe_dfma_tflops.restype = ctypes.c_double
    L.tccd_probe_dfma_tflops.argtypes = [ctypes.c_int, ctypes.c_int]
    L.tccd_probe_dadd_tflops.restype = ctypes.c_double
    L.tccd_probe_dadd_tflops.argtypes = [ctypes.c_int, ctypes.c_int]
    return {"dfma_tflops": L.tccd_probe_dfma_tflops(20000, 5),
            "dadd_tflops": L.tccd_probe_dadd_tflops(20000, 5)}


# ---------------------------------------------------------------------------
# the reference's CPU path (cpu_baseline and --impl reference)

def _numba_env():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tccd_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)


def reference_available() -> bool:
    try:
        _numba_env()
        import ccdkit._kernel  # noqa: F401
        return os.path.dirname(os.path.dirname(ccdkit._kernel.__file__)) == REF_DIR
    except Exception:
        return False


def _filters_np(pts: np.ndarray, kind: np.ndarray, sep: float) -> np.ndarray:
    """compute_gamma + compute_filters (inclusion.py:85-122) for a batch, in
    the reference's operation order: eps = coeff * (g * g * g)."""
    g = np.maximum(np.abs(pts).max(axis=1), 1.0)
    if sep > 0.0:
        coef = np.where(kind == 0, 7.549516567451064e-15, 7.105427357601002e-15)
    else:
        coef = np.where(kind == 0, 6.661338147750939e-15, 6.217248937900877e-15)
    return coef[:, None] * (g * g * g)


def _workloads_module():
    """workloads.py without the package __init__ (which imports torch): the
    spawn-pool workers stay light."""
    import importlib.util
    name = "_tccd_workloads"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(
        name, os.path.join(ROOT, "paper_2009_13349_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def _cpu_worker(job):
    """One spawn-pool worker: solve the blocks (w, w + W, ...) of the workload
    stream, query by query in its order, with the reference's numba kernel
    (or the C port) until its time is up."""
    cfg, sep, blocks, seconds, kind_of_run = job
    W = _workloads_module()
    if kind_of_run == "reference":
        _numba_env()
        from ccdkit import _kernel
        solve = _kernel.solve_kernel
        # (untimed: the first call loads the compiled kernel from numba's cache)
        solve(np.zeros((4, 3)), np.ones((4, 3)), 0, 1.0, 1e-6, 16, sep, 1e-14, 1e-14, 1e-14)
    else:
        sys.path.insert(0, ROOT)
        import oracle
        oracle.lib()
    done, t_used = 0, 0.0
    sub = 256
    for blk in blocks:
        if t_used >= seconds:
            break
        w = W.generate(cfg, blk * W.BLOCK, W.BLOCK, separation=sep)
        pts, kind = w.points, w.kind
        delta = np.broadcast_to(np.asarray(w.delta, dtype=np.float64), (w.n,))
        mc = np.broadcast_to(np.asarray(w.max_checks, dtype=np.int64), (w.n,))
        eps = _filters_np(pts, kind, sep)
        for a in range(0, w.n, sub):
            if t_used >= seconds:
                break
            b = min(w.n, a + sub)
            t0 = time.perf_counter()
            if kind_of_run == "reference":
                for i in range(a, b):
                    p = pts[i]
                    solve(p[:4], p[4:], int(kind[i]), 1.0, float(delta[i]), int(mc[i]), sep,
                          eps[i, 0], eps[i, 1], eps[i, 2])
            else:
                oracle.solve_batch(pts[a:b], kind[a:b], delta[a:b], mc[a:b], sep, 1.0, threads=1)
            t_used += time.perf_counter() - t0
            done += b - a
    return done, t_used


class CpuPath:
    """The reference's CPU path on all host cores (spawn pool, one worker per
    core in os.sched_getaffinity(0)), the pool started and JIT-warmed once."""

    def __init__(self, cfg: int, sep: float):
        import multiprocessing as mp
        self.cfg, self.sep = cfg, sep
        self.cores = len(os.sched_getaffinity(0))
        self.kind = "reference" if reference_available() else "port"
        if self.kind == "reference":
            # compile once here (numba cache=True), so the workers load it
            from ccdkit import _kernel
            _kernel.solve_kernel(np.zeros((4, 3)), np.ones((4, 3)), 0, 1.0, 1e-6, 16, sep,
                                 1e-14, 1e-14, 1e-14)
        self.pool = mp.get_context("spawn").Pool(self.cores)
        # warm every worker (imports, JIT cache load)
        self.pool.map(_cpu_worker, [(cfg, sep, [0], 0.0, self.kind)] * self.cores)

    def run(self, seconds: float) -> tuple[int, float]:
        """-> (queries solved, busy seconds of the slowest worker)."""
        W_ = self.cores
        jobs = [(self.cfg, self.sep, [w + W_ * k for k in range(10_000)], seconds, self.kind)
                for w in range(W_)]
        res = self.pool.map(_cpu_worker, jobs)
        return sum(r[0] for r in res), max(r[1] for r in res)

    def describe(self, n: int, t: float) -> str:
        what = ("ccdkit._kernel.solve_kernel (numba, baseline/_ref) called per query as "
                "ccdkit.solver.solve does, eps by compute_filters' formula"
                if self.kind == "reference"
                else "oracle/tccd_oracle.c (C restatement of the reference)")
        return (f"{n} queries: the leading queries of the workload's 65536-query blocks, "
                f"block b on worker b mod {self.cores} (spawn pool, one worker per core, "
                f"~{t:.1f}s busy each): {what}")

    def close(self):
        self.pool.terminate()


def solve_api_rate(cfg: int, sep: float, n: int = 2000) -> float | None:
    """ccdkit.solve() through the reference's public API on one core (Query
    objects, SolverConfig, the numba kernel) -- BASELINE.md §2."""
    try:
        _numba_env()
        from ccdkit import core, solver
        from paper_2009_13349_b200 import workloads as W
        w = W.generate(cfg, 0, n, separation=sep)
        qs = [core.Query(core.QueryKind(int(w.kind[i])), [tuple(r) for r in w.points[i, :4]],
                         [tuple(r) for r in w.points[i, 4:]]) for i in range(n)]
        conf = core.SolverConfig(separation=sep)
        solver.solve(qs[0], conf)
        t0 = time.perf_counter()
        for q in qs:
            solver.solve(q, conf)
        return n / (time.perf_counter() - t0)
    except Exception:
        return None


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    cpu = CpuPath(args.config, args.separation)
    for _ in range(args.warmup):
        cpu.run(0.3)
    total_q, total_t = 0, 0.0
    for s in range(args.steps):
        q, t = cpu.run(args.ref_step_seconds)
        total_q += q
        total_t += t
    cpu.close()
    value = total_q / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_desc(args.config, args.queries, args.gpus, args.separation),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cpu.cores, "kind": cpu.kind,
                         "sample": "each step: " + cpu.describe(total_q // args.steps,
                                                               total_t / args.steps)},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n: int) -> int:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def selftest_launcher(args, world: int, rank: int) -> None:
    """Launcher / sharding self-test for CPU-only machines (gloo): every rank
    takes its contiguous shard of the one set, the shards tile [0, Q), and
    rank 0 prints the line's n_gpus / scaling fields.  No solve runs."""
    import torch
    import torch.distributed as dist
    from paper_2009_13349_b200.solver import shard_bounds
    if world > 1:
        dist.init_process_group("gloo")
    lo, hi = shard_bounds(args.queries, world, rank)
    t = torch.tensor([lo, hi], dtype=torch.int64)
    parts = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    if world > 1:
        dist.all_gather(parts, t)
    else:
        parts = [t]
    if rank == 0:
        bounds = [tuple(int(x) for x in p) for p in parts]
        print(json.dumps({"n_gpus": world, "scaling": "strong", "queries": args.queries,
                          "shards": bounds}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def stage_flops(st: list, stage: str) -> float:
    """Algorithmic FP64 flops of one stage from the library's counters."""
    from paper_2009_13349_b200 import _lib as L
    if stage == "lane":
        return (st[L.STAT_LANE_CHECKS] * F_CHECK[0] + st[L.STAT_LANE_CHECKS + 1] * F_CHECK[1])
    if stage in ("light", "medium", "giant"):
        t = ("light", "medium", "giant").index(stage)
        vf, ee = st[L.STAT_CLS + 2 * t], st[L.STAT_CLS + 2 * t + 1]
        f = (vf * F_CHECK[0] + ee * F_CHECK[1]) / (vf + ee) if vf + ee else 0.0
        return st[L.STAT_TIER_CHECKS + t] * f
    return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--separation", type=float, default=0.0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--selftest-launcher", action="store_true",
                    help="CPU test of the N-rank launch and sharding only (gloo, no solve)")
    args = ap.parse_args()
    if args.queries is None:
        args.queries = DEFAULT_Q[args.config]

    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.impl == "ours" and world == 0 and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = max(world, 1)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.selftest_launcher:
        selftest_launcher(args, world, rank)
        return

    # this rank's contiguous shard of the one query set, generated before CUDA
    # is touched (forked workers)
    from paper_2009_13349_b200 import workloads as W
    from paper_2009_13349_b200.solver import shard_bounds
    Q = args.queries
    lo, hi = shard_bounds(Q, world, rank)
    t_gen = time.perf_counter()
    w = W.generate_parallel(args.config, lo, hi - lo, separation=args.separation,
                            workers=max(1, len(os.sched_getaffinity(0)) // world))
    t_gen = time.perf_counter() - t_gen

    import torch
    import torch.distributed as dist
    from paper_2009_13349_b200 import _lib, solve_batch, solver

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n = w.n
    pts_h = torch.from_numpy(w.points).pin_memory()
    kind_h = torch.from_numpy(w.kind).pin_memory()
    pts = pts_h.to(dev)
    kind = kind_h.to(dev)
    kw = {}
    if args.config == 2:
        kw = dict(delta=torch.from_numpy(w.delta).to(dev),
                  max_checks=torch.from_numpy(w.max_checks).to(dev))
    sep = args.separation
    stream = torch.cuda.current_stream(dev)
    flush = None
    if n * 192 <= 126e6:
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # the library records an event after every stage launch (prologue, lane,
    # then light / medium / giant per group-tier sub-chunk); stage times are
    # the gaps between consecutive events, summed per stage
    NEV = 256
    NS = len(solver.STAGES)

    def step(events=None, info=None):
        solve_batch(pts, kind, outputs=("status", "toi"), device=dev, separation=sep,
                    raise_on_error=False, info=info, events=events, **kw)

    # untimed: full outputs once, for the algorithmic work (checks), hits and
    # the library's per-stage counters
    full = solve_batch(pts, kind, device=dev, stats=True, separation=sep, raise_on_error=False, **kw)
    checks = full["checks"].cpu().numpy()
    status = full["status"].cpu().numpy()
    hits = int((status == 1).sum())
    valid = status < 2
    st = [int(x) for x in full["stats"].tolist()]
    vf = (w.kind == 0) & valid
    ee = (w.kind == 1) & valid
    flops = float(P_QUERY[0] * vf.sum() + P_QUERY[1] * ee.sum()
                  + F_CHECK[0] * checks[vf].sum() + F_CHECK[1] * checks[ee].sum())
    del full
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # per step: a start event + the library's stage events, all on the
    # launching stream; handles created here
    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(1 + NEV)] for _ in range(args.steps)]
    for row in sev:
        for ev in row:
            ev.record(stream)
    torch.cuda.synchronize(dev)
    infos = [{} for _ in range(args.steps)]
    if flush is None:
        e0.record(stream)
        for k in range(args.steps):
            sev[k][0].record(stream)
            step(sev[k][1:], infos[k])
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / args.steps
    else:
        for k in range(args.steps):
            flush.fill_(k & 255)
            sev[k][0].record(stream)
            step(sev[k][1:], infos[k])
        torch.cuda.synchronize(dev)
        ms = statistics.mean(sev[k][0].elapsed_time(sev[k][len(infos[k]["event_stages"])])
                             for k in range(args.steps))
    barrier()
    per = [solver.stage_times(sev[k][0], sev[k][1:], infos[k]["event_stages"])
           for k in range(args.steps)]
    stage_ms = {nm: statistics.mean(p[nm] for p in per) for nm in solver.STAGES}
    stage_launches = {nm: infos[0]["event_stages"].count(j) for j, nm in enumerate(solver.STAGES)}
    gpu_launches = sum(i["launches"] for i in infos)

    # end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        barrier()
        torch.cuda.synchronize(dev)
        kw_h = {k: v.cpu() for k, v in kw.items()}
        api = dict(outputs=(), hits=True, device=dev, non_blocking=True, separation=sep, **kw_h)
        # untimed warm-up with as many calls in flight as the timed loop has
        # (the caching allocators then hold every in-flight step's buffers)
        warm = [solve_batch(pts_h, kind_h, **api) for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        del warm
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        # the points copies run on the API's side stream, ordered after f0;
        # each chunk's solve waits for its own copy
        solver.copy_stream(dev).wait_event(f0)
        t_wall = time.perf_counter()
        infos = [{} for _ in range(args.steps)]
        res = [solve_batch(pts_h, kind_h, info=infos[k], **api) for k in range(args.steps)]
        f1.record(stream)  # after the last hit list's copy-out
        torch.cuda.synchronize(dev)
        t_wall = time.perf_counter() - t_wall
        counts = [int(r["hit_count"][0]) for r in res]
        assert all(c == hits for c in counts), "e2e hit lists differ from the device-input solve"
        got = np.sort(res[-1]["hit_index"][:hits].numpy())
        assert np.array_equal(got, np.flatnonzero(status == 1)), "e2e hit list differs"
        gpu_launches += sum(i["launches"] for i in infos)
        e2e_ms = f0.elapsed_time(f1) / args.steps
        e2e = {"ms": e2e_ms, "h2d": int(pts_h.numel() * 8 + kind_h.numel()),
               "d2h": int(hits * 16 + 8), "wall_ms": 1e3 * t_wall / args.steps}
        del res
    barrier()
    clk = clocks.stop()

    ms_max = max_over_ranks(ms)
    value = Q / (ms_max * 1e-3)
    e2e_value = None
    if e2e is not None:
        e2e_value = Q / (max_over_ranks(e2e["ms"]) * 1e-3)
    # rank-0 view of the aggregate counters (per-rank values are summed)
    def total(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t.item())
    hits_all = int(total(hits))
    flops_all = total(flops)
    launches_all = int(total(gpu_launches))
    if e2e is not None:
        e2e["h2d"] = int(total(e2e["h2d"]))
        e2e["d2h"] = int(total(e2e["d2h"]))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = fp64_peaks()
    dom = max(solver.STAGES, key=lambda nm: stage_ms[nm])
    dom_flops = stage_flops(st, dom)
    achieved = dom_flops / (stage_ms[dom] * 1e-3) / 1e12 if stage_ms[dom] > 0 else 0.0
    per_stage = {nm: {"ms": stage_ms[nm], "algorithmic_tflops":
                      stage_flops(st, nm) / (stage_ms[nm] * 1e-3) / 1e12 if stage_ms[nm] > 0.01
                      else None} for nm in solver.STAGES}
    traffic, ncu = None, None
    tpath = os.path.join(ROOT, "profiles", "r02", "roofline_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if tj.get("kernel") == dom and tj.get("config") == args.config:
            traffic = tj["dram_bytes_per_launch"]
            ncu = {k: tj[k] for k in ("fp64_pipe_active_pct", "warp_execution_efficiency_pct",
                                      "dram_gbs", "issue_slots_busy_pct", "source") if k in tj}
    cpu = None
    if not args.no_cpu:
        cp = CpuPath(args.config, sep)
        nq, t = cp.run(args.cpu_seconds)
        cp.close()
        cpu = {"value": nq / t, "unit": "queries/s", "cores": cp.cores, "kind": cp.kind,
               "sample": cp.describe(nq, t)}
        if cp.kind == "reference":
            r1 = solve_api_rate(args.config, sep)
            if r1:
                cpu["solve_api_single_core"] = {"value": r1, "unit": "queries/s",
                                                "sample": "2000 queries through ccdkit.solve()"}
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_2009_13349_b200/workloads.py)",
        "config": workload_desc(args.config, Q, world, sep),
        "e2e": None if e2e is None else {
            "value": e2e_value, "unit": "queries/s",
            "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
            "api": "solve_batch(pinned host points/kind, outputs=(), hits=True, "
                   "non_blocking=True): points H2D on the API's copy stream chunk by chunk "
                   "under the solve; the compacted hit list (index, toi) and its count D2H by "
                   "a copy-out kernel moving only live entries; CUDA events on the launching "
                   "stream, max over ranks",
            "wall_ms_per_step_rank0": e2e["wall_ms"]},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peaks["dfma_tflops"],
                     "unit": "TFLOP/s", "frac": achieved / peaks["dfma_tflops"],
                     "traffic": traffic,
                     "kernel": KERNEL_NAMES[dom],
                     "kernel_flops_per_launch": dom_flops / max(stage_launches[dom], 1),
                     "kernel_ms_per_launch": stage_ms[dom] / max(stage_launches[dom], 1),
                     "launches_per_step": stage_launches[dom],
                     "share_of_step": stage_ms[dom] / ms,
                     "stages": per_stage,
                     "peak_source": "measured on this box: DFMA probe (libtccd_probe.so), "
                                    "FMA-counted (2 flops per DFMA)",
                     "fma_free_ceiling_tflops": peaks["dadd_tflops"],
                     "frac_of_fma_free_ceiling": achieved / peaks["dadd_tflops"],
                     "solve_flops_per_step": flops_all,
                     "solve_achieved_tflops": flops_all / (ms_max * 1e-3) / 1e12,
                     "traffic_source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum"
                                       " (profiles/r02/roofline_traffic.json)" if traffic else None,
                     "ncu_counters": ncu},
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": launches_all,
        "workload_stats": {
            "hits": hits_all, "hit_rate": hits_all / Q, "rank0_mean_checks": float(checks.mean()),
            "rank0_max_checks": int(checks.max()), "rank0_stats": {
                "decided_at_root": st[_lib.STAT_PROLOGUE_DONE],
                "lane_queries": st[_lib.STAT_LANE_QUERIES],
                "lane_finished": st[_lib.STAT_LANE_DONE] + st[_lib.STAT_LANE_DONE + 1],
                "lane_evicted": st[_lib.STAT_LANE_EVICTED],
                "lane_wasted_checks": st[_lib.STAT_LANE_WASTED],
                "medium_tier_queries": st[_lib.STAT_MEDIUM_QUERIES],
                "giant_tier_queries": st[_lib.STAT_GIANT_QUERIES],
                "handover_restarts": st[_lib.STAT_RESTARTS:_lib.STAT_RESTARTS + 2],
                "group_tier_path_checks": st[_lib.STAT_TIER_CHECKS:_lib.STAT_TIER_CHECKS + 3],
                "group_tier_classifications": st[_lib.STAT_CLS:_lib.STAT_CLS + 6]},
            "generation_s_rank0": t_gen},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
