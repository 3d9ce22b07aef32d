"""Host-side logic of the multi-GPU path, on CPU with gloo (world_size 2).

The device data path (in-kernel replicated stores + cross-shard barrier) is
covered on one GPU by tests/test_gpu_parity.py::test_virtual_shards_*; here
the torch.distributed plumbing around it runs for real in two processes:
handle exchange, objective/edge reduction, Omega column gather, partition.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2106_09382_b200 import dist as cdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. IPC handle all-gather: fixed-size, rank order
        h = bytes([rank + 1]) * 64
        allh = cdist.exchange_handles(h)
        # 2. per-sweep objective partials + edge count summed over shards
        parts = np.arange(7, dtype=np.float64) * (rank + 1)
        tot = cdist.reduce_parts(parts)
        # 3. Omega assembled from column blocks (uneven split, last shard smaller)
        p = 11
        full = np.arange(p * p, dtype=np.float64).reshape(p, p)
        ranges = [(0, 6), (6, 11)]
        c0, c1 = ranges[rank]
        got = cdist.gather_columns(full[:, c0:c1], c0, p)
        got0 = cdist.gather_columns(full[:, c0:c1], c0, p, dst=0)
        results[rank] = (allh, tot.tolist(), bool(np.array_equal(got, full)),
                         None if got0 is None else bool(np.array_equal(got0, full)))
    finally:
        dist.destroy_process_group()


def test_host_plumbing_two_ranks_gloo():
    world = 2
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
        res = dict(results)
    want_h = bytes([1]) * 64 + bytes([2]) * 64
    for r in range(world):
        allh, tot, ok, ok0 = res[r]
        assert allh == want_h
        assert tot == (np.arange(7.0) * 3).tolist()
        assert ok
    assert res[0][3] is True and res[1][3] is None


@pytest.mark.parametrize("p", [100, 1000, 5000, 20000, 50000])
@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_partition_covers_columns_once(p, g):
    part = cdist.partition(p, g, rank=0 if g > 1 else None)
    cols = [c for a, b in part["ranges"] for c in range(a, b)]
    assert cols == list(range(p))
    assert part["slab_width"] % 2 == 0
    assert part["blocks_total"] == part["blocks_per_shard"] * g


def test_objective_from_parts_matches_model_formula():
    parts = np.array([[10.0, 2.0, 0.5], [8.0, 1.0, 0.25]])
    n, lam = 50.0, 0.3
    want = [-n * 0.5 + 5.0 + n * lam * 2.0, -n * 0.25 + 4.0 + n * lam * 1.0]
    np.testing.assert_allclose(cdist.objective_from_parts(parts, n, lam), want)
