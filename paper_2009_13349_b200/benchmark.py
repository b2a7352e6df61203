"""Benchmark harness on the GPU batch: verdicts vs labels, FP/FN accounting.

Mirrors the reference harness (pkg/src/ccdkit/bench.py:49-259) for the
"ours" method and the "irf" interval baseline (both on the GPU; the
univariate cubic baseline is not provided): a method's verdict on a query
is its collision flag;
against ground truth this yields false positive / false negative /
correct / undecided counts, plus budget-ended (early) solves.  The
reference times each query with a nanosecond clock around ``solve``; here a
whole labeled set is one batched call, timed with CUDA events on the
launching stream after a warm-up solve, so ``avg_time_us`` is batch time /
queries (a throughput figure, not a per-query latency) and the histogram
is of per-query check counts, binned like the reference's runtime bins.
Filter resolution happens on the device inside the timed call (the
reference precomputes it outside its timed region, bench.py:152-160).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .baselines import irf_batch
from .core import SolverConfig
from .dataset import LabeledBatch
from .solver import solve_batch

METHOD_NAMES = ("ours", "irf")  # the reference's order (bench.py:43), univariate not provided

# checks histogram: 24 log-spaced bins from 1 to 10^6 (out of range clamps)
HIST_EDGES_CHECKS = tuple(float(x) for x in np.logspace(0.0, 6.0, 25))


@dataclass(frozen=True)
class MethodStats:
    name: str
    avg_time_us: float
    fp_count: int
    fn_count: int
    correct_count: int
    undecided_count: int
    early_count: int
    histogram: tuple
    verdicts: tuple

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        d["histogram"] = list(self.histogram)
        d["verdicts"] = [int(v) for v in self.verdicts]
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "MethodStats":
        return cls(d["name"], d["avg_time_us"], d["fp_count"], d["fn_count"],
                   d["correct_count"], d["undecided_count"], d["early_count"],
                   tuple(d["histogram"]), tuple(bool(v) for v in d["verdicts"]))


@dataclass(frozen=True)
class BenchReport:
    methods: tuple
    size: int
    delta: float
    max_checks: int
    separation: float
    t_max: float
    seed: int | None
    queries_per_second: float
    histogram_edges_checks: tuple = HIST_EDGES_CHECKS

    def method(self, name: str) -> MethodStats:
        for m in self.methods:
            if m.name == name:
                return m
        raise KeyError(name)

    def to_dict(self) -> dict:
        return {"methods": [m.to_dict() for m in self.methods], "size": self.size,
                "delta": self.delta, "max_checks": self.max_checks,
                "separation": self.separation, "t_max": self.t_max, "seed": self.seed,
                "queries_per_second": self.queries_per_second,
                "histogram_edges_checks": list(self.histogram_edges_checks)}

    @classmethod
    def from_dict(cls, d: dict) -> "BenchReport":
        return cls(tuple(MethodStats.from_dict(m) for m in d["methods"]), d["size"], d["delta"],
                   d["max_checks"], d["separation"], d["t_max"], d["seed"],
                   d["queries_per_second"], tuple(d["histogram_edges_checks"]))


def _normalize_methods(methods) -> tuple:
    """bench.py:139-149: lower-cased, de-duplicated, in METHOD_NAMES order."""
    if isinstance(methods, str):
        methods = (methods,)
    chosen = []
    for m in methods:
        name = str(m).strip().lower()
        if name not in METHOD_NAMES:
            raise ValueError(f"unknown method {m!r}; expected one of {METHOD_NAMES}")
        if name not in chosen:
            chosen.append(name)
    if not chosen:
        raise ValueError("no methods selected")
    return tuple(sorted(chosen, key=METHOD_NAMES.index))


def run_benchmark(data: LabeledBatch, methods=("ours",), cfg: SolverConfig | None = None, *,
                  seed=None, device=None, repeats: int = 1) -> BenchReport:
    """Run each selected method ("ours", "irf") over every query of a labeled
    batch on the GPU and score verdicts (bench.py:192-259).  IRF uses the
    config's delta, max_checks and t_max (bench.py:169-175)."""
    cfg = cfg or SolverConfig()
    names = _normalize_methods(methods)
    n = data.n
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if n == 0:
        empty = tuple(MethodStats(nm, 0.0, 0, 0, 0, 0, 0, (0,) * 24, ()) for nm in names)
        return BenchReport(empty, 0, cfg.delta, cfg.max_checks, cfg.separation, cfg.t_max,
                           seed, 0.0)
    pts = torch.from_numpy(np.ascontiguousarray(data.points)).to(dev)
    kind = torch.from_numpy(np.ascontiguousarray(data.kind)).to(dev)
    truth = np.asarray(data.truth)
    decided = truth >= 0
    stream = torch.cuda.current_stream(dev)
    stats, qps = [], None
    for name in names:
        if name == "ours":
            def run(p, k):
                return solve_batch(p, k, cfg, outputs=("status", "toi", "checks", "early"),
                                   device=dev, raise_on_error=True)
        else:
            def run(p, k):
                return irf_batch(p, k, cfg.delta, cfg.max_checks, cfg.t_max, device=dev)
        run(pts[:1], kind[:1])  # warm-up (excluded)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(repeats):
            res = run(pts, kind)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / repeats
        verdict = (res["status"] == 1).cpu().numpy()
        early = res["early"].cpu().numpy().astype(bool)
        checks = res["checks"].cpu().numpy()
        fp = int(np.sum(decided & verdict & (truth == 0)))
        fn = int(np.sum(decided & ~verdict & (truth == 1)))
        undecided = int(np.sum(~decided))
        correct = n - fp - fn - undecided
        clipped = np.clip(checks.astype(np.float64), HIST_EDGES_CHECKS[0], HIST_EDGES_CHECKS[-1])
        hist, _ = np.histogram(clipped, bins=np.asarray(HIST_EDGES_CHECKS))
        stats.append(MethodStats(name, ms * 1e3 / n, fp, fn, correct, undecided, int(early.sum()),
                                 tuple(int(h) for h in hist), tuple(bool(v) for v in verdict)))
        if qps is None:
            qps = n / (ms * 1e-3)
    return BenchReport(tuple(stats), n, cfg.delta, cfg.max_checks, cfg.separation, cfg.t_max,
                       seed, qps)


_CSV_FIELDS = ("name", "avg_time_us", "fp_count", "fn_count", "correct_count",
               "undecided_count", "early_count")


def format_report(report: BenchReport, format: str) -> str:
    if format == "json":
        return json.dumps(report.to_dict(), sort_keys=True, indent=2) + "\n"
    if format == "csv":
        lines = [",".join(_CSV_FIELDS)]
        for m in report.methods:
            d = m.to_dict()
            lines.append(",".join(str(d[f]) for f in _CSV_FIELDS))
        return "\n".join(lines) + "\n"
    raise ValueError("format must be 'json' or 'csv'")


def emit_report(report: BenchReport, format: str, path) -> None:
    Path(path).write_text(format_report(report, format), encoding="ascii")


def load_report(path) -> BenchReport:
    return BenchReport.from_dict(json.loads(Path(path).read_text(encoding="ascii")))
