"""Small batches through every kernel of the library.

Run it against the bounds-checked build of the library (every index written
by the engine asserted against its array's capacity; a violation traps):

    (cd paper_2009_13349_b200/csrc && nvcc <Makefile flags> --fmad=false -DTCCD_CHECKS \
        -shared -o ../../exp/lib_checks.so tccd.cu broad.cu irf.cu)
    TCCD_LIB=exp/lib_checks.so python tools/sanitize.py

or under compute-sanitizer where it is available (memcheck, racecheck with
--quick).

Covers: prologue, lane tier, light / medium / giant engine tiers (mixed
batch; giant alone), the general (non-dyadic t_max) ordering path, minimum separation,
per-query delta / max_checks, the IRF baseline's three passes and the GPU
broad phase.  Every solver result is checked bit for bit against the oracle
(test infrastructure), so a run that exits 0 is also a parity pass.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2009_13349_b200 import solve_batch  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402
from paper_2009_13349_b200.baselines import irf_batch  # noqa: E402
from paper_2009_13349_b200.scene import TriMeshPair, broad_phase_batch  # noqa: E402

FIELDS = ("status", "toi", "tol", "codom", "checks", "early", "witness", "level")


def same(got, ref, what):
    for k in FIELDS:
        a = got[k].cpu().numpy()
        b = ref[k]
        ok = np.array_equal(a.view(np.int64), b.view(np.int64)) if a.dtype.kind == "f" else \
            np.array_equal(a, b)
        if not ok:
            raise SystemExit(f"{what}: field {k} differs from the oracle")
    print(f"ok {what}: {len(ref['status'])} queries, {int(ref['checks'].sum())} checks", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="smaller batches (racecheck is slow)")
    args = ap.parse_args()
    s = 4 if args.quick else 1
    dev = torch.device("cuda", 0)
    mc = 20_000 // s

    def run(cfg, start, n, what, **kw):
        w = W.generate(cfg, start, n, separation=kw.pop("sep", None))
        d = w.delta if cfg == 2 else 1e-6
        m = np.minimum(w.max_checks, mc) if cfg == 2 else mc
        tm = kw.pop("t_max", 1.0)
        got = solve_batch(torch.from_numpy(w.points).to(dev), torch.from_numpy(w.kind).to(dev),
                          delta=torch.as_tensor(d).to(dev) if cfg == 2 else d,
                          max_checks=torch.as_tensor(m).to(dev) if cfg == 2 else m,
                          separation=w.separation, t_max=tm, device=dev, raise_on_error=False,
                          **kw)
        ref = oracle.solve_batch(w.points, w.kind, d, m, w.separation, tm)
        same(got, ref, what)

    run(3, 0, 8192 // s, "config 3 (lane tier, handovers)")
    run(1, 0, 2048 // s, "config 1 (light / medium / giant)")
    run(0, 5000, 1024 // s, "config 0")
    run(2, 0, 256 // s, "config 2 (per-query delta / max_checks)")
    run(1, 7000, 512 // s, "config 1 at t_max = 0.7 (general ordering)", t_max=0.7)
    run(4, 0, 128 // s, "config 4 at d = 1e-5", sep=1e-5)
    run(1, 3000, 256 // s, "config 1, giant tier alone", heavy_only=True)

    w = W.generate(1, 100, 512 // s)
    pts, kind = torch.from_numpy(w.points).to(dev), torch.from_numpy(w.kind).to(dev)
    ref = oracle.irf_batch(w.points, w.kind, 1e-6, 5000 // s, 1.0)
    same(irf_batch(pts, kind, 1e-6, 5000 // s, 1.0, device=dev), ref, "IRF passes 1 + 2")
    same(irf_batch(pts, kind, 1e-6, 5000 // s, 1.0, device=dev, heavy_only=True), ref,
         "IRF pass 2 alone")

    rng = np.random.default_rng(7)
    g = 12
    xs, ys = np.meshgrid(np.linspace(0, 1, g), np.linspace(0, 1, g))
    x0 = np.stack([xs.ravel(), ys.ravel(), np.zeros(g * g)], 1)
    tris = [(i * g + j, i * g + j + 1, (i + 1) * g + j) for i in range(g - 1) for j in range(g - 1)]
    x1 = x0 + rng.normal(0, 0.05, x0.shape)
    cs = broad_phase_batch(TriMeshPair(x0, x1, np.array(tris)), 0.01, device=dev)
    torch.cuda.synchronize()
    print(f"ok broad phase: {len(cs.kind)} candidates", flush=True)


if __name__ == "__main__":
    main()
