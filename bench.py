"""Benchmark: CCD queries/sec (FP64, delta=1e-6) on B200, + FP64 roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1] [--queries Q]

One step = one batched solve of this rank's queries of the workload (default
BASELINE config 1: mixed VF/EE, half planted collisions, delta=1e-6,
m_I=1e6, d=0, t_max=1; Q = 10^6 queries per GPU, weak scaling: rank r solves
queries [r*Q, (r+1)*Q) of the index-addressable synthetic stream).  Inputs
(192 MB per 10^6 queries) exceed the 126 MB L2, so no flush is needed.

value  = device-timed throughput, inputs resident in HBM, CUDA events on the
         launching stream, barrier + synchronize on both sides, max over ranks.
e2e    = the same through the public API with pinned HOST inputs: H2D of
         points + kind and D2H of status + toi inside the timed region.
roofline = the dominant kernel (the light-tier engine_kernel): its
         algorithmic FP64 flops per launch (F_VF = 200 / F_EE = 174
         per box classification, counted per tier and kind by the library) /
         its average duration, timed with CUDA events the library records on
         the launching stream after every stage of every timed step; peak =
         the DFMA rate measured on this box by libtccd_probe.so (FMA-counted;
         an FMA-free kernel is capped at 0.5 of it).  traffic = that kernel's
         DRAM bytes per launch from the committed ncu capture
         (profiles/r01/roofline_traffic.json).
cpu_baseline = the C restatement of the reference (oracle/, kind "port") on
         all host cores, rank 0 at N=1, on a bounded sample.
--impl reference: that CPU path alone, same metric/config (rank 0 only).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
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
LAUNCHES_PER_SOLVE = 5  # per 2^22-query chunk: prologue, light, medium, giant-queue order, giant


def algorithmic_flops(kind: np.ndarray, checks: np.ndarray) -> float:
    vf = kind == 0
    return float(np.sum(np.where(vf, P_QUERY[0] + checks * F_CHECK[0],
                                 P_QUERY[1] + checks * F_CHECK[1]).astype(np.float64)))


def workload_desc(cfg: int, q: int) -> dict:
    from paper_2009_13349_b200 import workloads as W
    names = {
        0: "config0: vertex-face, U[0,1]^3 + U[-0.5,0.5]^3 motion",
        1: "config1: 50% VF / 50% EE, half planted exact roots, half config-0 random",
        2: "config2: degenerate lattice families, delta in {1e-4,1e-6,1e-8}, m_I in {1e3,1e6}",
        3: "config3: simulation-shaped, 80% VF / 20% EE, edge 1e-2, offsets N(0,1e-3)/N(0,5e-3)",
    }
    return {"workload": names.get(cfg, W.CONFIGS[cfg]["name"]), "baseline_config": cfg,
            "queries_per_gpu": q, "delta": 1e-6 if cfg != 2 else "per-query",
            "max_checks": 1_000_000 if cfg != 2 else "per-query", "separation": 0.0,
            "t_max": 1.0, "seed": f"PCG64(SeedSequence([{W.SEED_BASE}+{cfg}, block]))",
            "l2": "inputs > 126 MB L2 per step (no flush needed)" if q * 192 > 126e6
            else "inputs < L2; L2 flushed between steps"}


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
    so = os.path.join(ROOT, "paper_2009_13349_b200", "libtccd_probe.so")
    L = ctypes.CDLL(so)
    L.tccd_probe_dfma_tflops.restype = ctypes.c_double
    L.tccd_probe_dfma_tflops.argtypes = [ctypes.c_int, ctypes.c_int]
    L.tccd_probe_dadd_tflops.restype = ctypes.c_double
    L.tccd_probe_dadd_tflops.argtypes = [ctypes.c_int, ctypes.c_int]
    return {"dfma_tflops": L.tccd_probe_dfma_tflops(20000, 5),
            "dadd_tflops": L.tccd_probe_dadd_tflops(20000, 5)}


def cpu_sample(cfg: int, start: int, target_s: float, threads: int, chunk: int = 20000):
    """Run the oracle port on consecutive chunks until ~target_s elapsed."""
    import oracle
    from paper_2009_13349_b200 import workloads as W
    done, t_cpu, lo = 0, 0.0, start
    while t_cpu < target_s:
        w = W.generate(cfg, lo, chunk)
        t0 = time.perf_counter()
        oracle.solve_batch(w.points, w.kind, w.delta, w.max_checks, w.separation, w.t_max,
                           threads=threads)
        t_cpu += time.perf_counter() - t0
        done += w.n
        lo += w.n
    return done, t_cpu


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    import oracle
    oracle.lib()
    per_step = max(args.ref_step_seconds, 0.5)
    for _ in range(args.warmup):
        cpu_sample(args.config, 0, 0.2, threads)
    total_q, total_t = 0, 0.0
    for s in range(args.steps):
        q, t = cpu_sample(args.config, s * 200_000, per_step, threads)
        total_q += q
        total_t += t
    value = total_q / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_desc(args.config, args.queries),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "port",
                         "sample": f"{total_q} queries of the workload stream in {args.steps} "
                                   f"steps of ~{per_step:.0f}s (oracle/tccd_oracle.c, pthreads)"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--queries", type=int, default=1_000_000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2009_13349_b200 import solve_batch, solver
    from paper_2009_13349_b200 import workloads as W

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

    Q = args.queries
    w = W.generate(args.config, rank * Q, Q)
    pts_h = torch.from_numpy(w.points).pin_memory()
    kind_h = torch.from_numpy(w.kind).pin_memory()
    pts = pts_h.to(dev)
    kind = kind_h.to(dev)
    kw = {}
    if args.config == 2:
        kw = dict(delta=torch.from_numpy(w.delta).to(dev), max_checks=torch.from_numpy(w.max_checks).to(dev))
    stream = torch.cuda.current_stream(dev)

    # the library solves a batch in 2^22-query chunks and records its stage
    # events once per chunk; a multi-chunk step is issued chunk by chunk here
    # (the same kernels on the same stream) so that every chunk's stages are
    # timed and summed
    CH = 1 << 22
    nch = (Q + CH - 1) // CH

    def step(events=None):
        for j in range(nch):
            lo, hi = j * CH, min(Q, (j + 1) * CH)
            kj = {k: v[lo:hi] for k, v in kw.items()}
            solve_batch(pts[lo:hi], kind[lo:hi], outputs=("status", "toi"), device=dev,
                        raise_on_error=False,
                        events=events[4 * j:4 * j + 4] if events else None, **kj)

    # untimed: full outputs once, for the algorithmic work (checks) and hits
    full = solve_batch(pts, kind, device=dev, stats=True, **kw)
    checks = full["checks"].cpu().numpy()
    hits = int((full["status"] == 1).sum().item())
    evicted = int(full["stats"][0].item())  # queries that reached the giant tier
    pool_rounds = int(full["stats"][1].item())
    deferrals = int(full["stats"][2].item())
    flops = algorithmic_flops(w.kind, checks)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # per step: solve start + the library's 4 stage events (prologue, light,
    # medium, giant done), all on the launching stream; handles created here
    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(1 + 4 * nch)]
           for _ in range(args.steps)]
    for row in sev:
        for ev in row:
            ev.record(stream)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for k in range(args.steps):
        sev[k][0].record(stream)
        step(sev[k][1:])
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    stage_names = ("prologue", "light", "medium", "giant")
    # stage j of chunk c runs from event 4c + j to 4c + j + 1 (event 0: step start)
    stage_ms = {nm: statistics.mean(sum(sev[k][4 * c + j].elapsed_time(sev[k][4 * c + j + 1])
                                        for c in range(nch)) for k in range(args.steps))
                for j, nm in enumerate(stage_names)}
    # end to end through the public API with pinned host buffers
    barrier()
    torch.cuda.synchronize(dev)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kw_h = {k: v.cpu() for k, v in kw.items()}
    # untimed warm-up of this path, with as many calls in flight as the timed
    # loop has (creates the API's copy stream; the caching allocators then
    # hold the device copies and pinned result buffers of every in-flight
    # step, so no cudaMalloc / cudaHostAlloc synchronizes the timed region)
    warm = [solve_batch(pts_h, kind_h, outputs=("status", "toi"), device=dev, non_blocking=True,
                        **kw_h) for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    del warm
    f0.record(stream)
    # the points copies run on the API's side stream, ordered after f0; each
    # solve waits for its copy, so step k+1's copy overlaps step k's solve
    solver.copy_stream(dev).wait_event(f0)
    t_wall = time.perf_counter()
    res = [solve_batch(pts_h, kind_h, outputs=("status", "toi"), device=dev, non_blocking=True,
                       **kw_h) for _ in range(args.steps)]
    f1.record(stream)  # after the last results' D2H
    torch.cuda.synchronize(dev)
    t_wall = time.perf_counter() - t_wall
    e2e_hits = [int((r["status"] == 1).sum()) for r in res]
    assert all(h == hits for h in e2e_hits), "e2e results differ from the device-input solve"
    barrier()
    clk = clocks.stop()
    e2e_ms = f0.elapsed_time(f1) / args.steps

    ms_max = max_over_ranks(ms)
    e2e_ms_max = max_over_ranks(e2e_ms)
    total_q = Q * world
    value = total_q / (ms_max * 1e-3)
    e2e_value = total_q / (e2e_ms_max * 1e-3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = fp64_peaks()
    st = [int(x) for x in full["stats"].tolist()]
    tier_flops = {nm: st[8 + 2 * t] * F_CHECK[0] + st[9 + 2 * t] * F_CHECK[1]
                  for t, nm in enumerate(("light", "medium", "giant"))}
    dom = max(("light", "medium", "giant"), key=lambda nm: stage_ms[nm])
    achieved = tier_flops[dom] / (stage_ms[dom] * 1e-3) / 1e12
    traffic = None
    ncu_counters = None
    tpath = os.path.join(ROOT, "profiles", "r01", "roofline_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if tj.get("kernel") == dom and tj.get("config") == args.config and tj.get("queries") == Q:
            traffic = tj["dram_bytes_per_launch"]
            ncu_counters = {k: tj[k] for k in ("fp64_pipe_active_pct", "warp_execution_efficiency_pct",
                                               "dram_gbs", "issue_slots_busy_pct") if k in tj}
    cpu = None
    if world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        nq, t = cpu_sample(args.config, 0, args.cpu_seconds, threads)
        cpu = {"value": nq / t, "unit": "queries/s", "cores": threads, "kind": "port",
               "sample": f"first {nq} queries of the same workload stream "
                         f"(oracle/tccd_oracle.c on {threads} threads, {t:.1f}s)"}
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_2009_13349_b200/workloads.py)",
        "config": workload_desc(args.config, Q),
        "e2e": {"value": e2e_value, "unit": "queries/s",
                "h2d_bytes_per_step": int(pts_h.numel() * 8 + kind_h.numel()),
                "d2h_bytes_per_step": int(Q * 9),
                "api": "solve_batch(pinned host points/kind, non_blocking=True): points H2D on "
                       "the API's copy stream (overlaps the previous step's solve), status+toi "
                       "D2H into pinned host tensors; CUDA events on the launching stream",
                "wall_ms_per_step": 1e3 * t_wall / args.steps},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peaks["dfma_tflops"],
                     "unit": "TFLOP/s", "frac": achieved / peaks["dfma_tflops"],
                     "traffic": traffic,
                     "kernel": f"engine_kernel ({dom} tier)",
                     "kernel_flops_per_launch": tier_flops[dom],
                     "kernel_ms": stage_ms[dom],
                     "share_of_step": stage_ms[dom] / ms,
                     "stage_ms": stage_ms,
                     "peak_source": "measured on this box: DFMA probe (libtccd_probe.so), FMA-counted",
                     "fma_free_ceiling_tflops": peaks["dadd_tflops"],
                     "frac_of_fma_free_ceiling": achieved / peaks["dadd_tflops"],
                     "solve_flops_per_step": flops,
                     "solve_achieved_tflops": flops / (ms * 1e-3) / 1e12,
                     "traffic_source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum"
                                       " (profiles/r01/roofline_traffic.json)",
                     "ncu_counters": ncu_counters},
        "cpu_baseline": cpu,
        "clocks": clk,
        # timed device steps + timed e2e steps (whose two result copy-outs,
        # status and toi, are kernels too)
        "gpu_launches": args.steps * LAUNCHES_PER_SOLVE * nch
                        + args.steps * (LAUNCHES_PER_SOLVE * nch + 2),
        "workload_stats": {"hits": hits, "hit_rate": hits / Q, "mean_checks": float(checks.mean()),
                           "max_checks": int(checks.max()), "giant_tier_queries": evicted,
                           "engine_rounds": pool_rounds, "level_deferrals": deferrals,
                           "medium_tier_queries": int(full["stats"][3].item()),
                           "boxes_per_tier": st[4:7],
                           "classifications_per_tier_vf_ee": [st[8:10], st[10:12], st[12:14]]},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
