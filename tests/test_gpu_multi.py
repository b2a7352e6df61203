"""GPU: several devices from one process (solve_devices) and one process per
device (solve_sharded, gloo gather), both through the product solve, against
the oracle.  The box has one GPU, so the same device appears in every shard
(the shards then share its workspace; the code path is the multi-device one).
"""

import os

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_same_results

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,count,devices", [(3, 300_001, [0, 0]), (1, 20_000, [0, 0, 0]),
                                                  (0, 10_000, [0])])
def test_solve_devices_matches_oracle(cuda, config, count, devices):
    from paper_2009_13349_b200 import solve_devices
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, 5_000, count)
    ref = oracle.solve_batch(w.points, w.kind)
    got = solve_devices(w.points, w.kind, devices, outputs=("status", "toi", "tol", "codom",
                                                            "checks", "early", "witness", "level"),
                        hits=True)
    assert_same_results({k: v.numpy() for k, v in got.items() if not k.startswith("hit_")}, ref,
                        f"solve_devices c{config}")
    hit = np.flatnonzero(ref["status"] == 1)
    order = np.argsort(got["hit_index"].numpy())
    assert np.array_equal(got["hit_index"].numpy()[order], hit)
    assert np.array_equal(got["hit_toi"].numpy()[order].view(np.int64), ref["toi"][hit].view(np.int64))


def test_solve_devices_per_query_parameters(cuda):
    from paper_2009_13349_b200 import solve_devices
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(2, 1_000, 3_000)
    ref = oracle.solve_batch(w.points, w.kind, w.delta, w.max_checks)
    got = solve_devices(w.points, w.kind, [0, 0], delta=w.delta, max_checks=w.max_checks,
                        outputs=("status", "toi", "checks"))
    assert_same_results({k: v.numpy() for k, v in got.items()}, ref, "per-query params")


def _rank(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200.sharding import solve_sharded
    from paper_2009_13349_b200 import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    w = W.generate(3, 0, 200_003)
    res = solve_sharded(w.points, w.kind,
                        lambda p, k, **kw: solve_batch(torch.from_numpy(np.ascontiguousarray(p)),
                                                       torch.from_numpy(np.ascontiguousarray(k)),
                                                       device=dev, raise_on_error=False),
                        rank=rank, world=world)
    if rank == 0:
        np.savez(out_path, **res)
    dist.destroy_process_group()


def test_solve_sharded_two_ranks_product_solve(cuda, tmp_path):
    import socket
    import torch.multiprocessing as mp
    from paper_2009_13349_b200 import workloads as W
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "r.npz")
    mp.spawn(_rank, args=(2, port, out), nprocs=2, join=True)
    got = dict(np.load(out))
    w = W.generate(3, 0, 200_003)
    ref = oracle.solve_batch(w.points, w.kind)
    assert_same_results(got, ref, "solve_sharded x2")
