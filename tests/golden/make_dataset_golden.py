"""Golden files for the dataset format and the benchmark harness.

Runs the REFERENCE (ccdkit, imported from /root/reference in the build
container) to produce, per kind:
  * ``ds_<set>_<kind>.csv`` -- its ``write_queries`` output
    (pkg/src/ccdkit/dataset.py:227-250) for the handcrafted battery and a
    seeded adversarial random set (planted roots + oracle-certified misses);
  * ``ds_<set>_<kind>.npz`` -- what its ``parse_queries`` (:168-199) makes of
    that file (binary64 coordinates, truth) and the verdicts and FP/FN counts
    of its ``run_benchmark(..., ("ours",))`` (pkg/src/ccdkit/bench.py:192).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_dataset_golden.py
"""

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from ccdkit import QueryKind, gen_handcrafted, gen_random  # noqa: E402
from ccdkit.bench import run_benchmark  # noqa: E402
from ccdkit.dataset import Profile, parse_queries, write_queries  # noqa: E402


def main():
    sets = {
        "handcrafted": lambda k: [lq for lq in gen_handcrafted() if lq.kind is k],
        "adv": lambda k: gen_random(30, seed=7 + int(k), profile=Profile.ADVERSARIAL,
                                    positive_fraction=0.5, kind=k)[0],
    }
    for name, make in sets.items():
        for k, tag in ((QueryKind.VERTEX_FACE, "vf"), (QueryKind.EDGE_EDGE, "ee")):
            qs = make(k)
            path = os.path.join(HERE, f"ds_{name}_{tag}.csv")
            write_queries(qs, path)
            parsed = parse_queries(path, k)
            pts = np.array([lq.query.all_coordinates() for lq in parsed])
            truth = np.array([lq.truth for lq in parsed], dtype=np.int8)
            rep = run_benchmark(parsed, ("ours",))
            m = rep.method("ours")
            np.savez_compressed(os.path.join(HERE, f"ds_{name}_{tag}.npz"), points=pts,
                                truth=truth, verdicts=np.array(m.verdicts, dtype=bool),
                                fp=m.fp_count, fn=m.fn_count, correct=m.correct_count,
                                early=m.early_count)
            print(name, tag, len(qs), "fp", m.fp_count, "fn", m.fn_count, "early", m.early_count)


if __name__ == "__main__":
    main()
