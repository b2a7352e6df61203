"""How many batched solves a line_search_step issues (each alpha-lowering
re-solves the remaining candidates at the new alpha) and how many candidate
solves in total, on the synthetic cloth scene of tools/scene_bench.py.

    python tools/ls_probe.py [--grid 100]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from scene_bench import cloth  # noqa: E402

import paper_2009_13349_b200.scene as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=100)
args = ap.parse_args()
calls = []
orig = S._solve


def counted(cs, sel, cfg, separation, device):
    t0 = time.perf_counter()
    r = orig(cs, sel, cfg, separation, device)
    calls.append((len(r["status"]), time.perf_counter() - t0))
    return r


S._solve = counted
mesh = cloth(args.grid)
t0 = time.perf_counter()
ls = S.line_search_step(mesh, p=0.5)
t = time.perf_counter() - t0
print(f"grid {args.grid}: {t * 1e3:.0f} ms, {len(ls.bounds)} bounds, {len(calls)} solves, "
      f"{sum(c[0] for c in calls)} candidate solves, solve time {sum(c[1] for c in calls) * 1e3:.0f} ms")

# second (warm) call under cProfile
import cProfile  # noqa: E402
import pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
S.line_search_step(mesh, p=0.5)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
