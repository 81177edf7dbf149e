"""Multi-rank host logic of the column-block sharding on CPU with gloo,
world_size 2: each rank computes its shard's product with the C oracle (standing in for
its GPU), the slices are all-gathered, and the result must equal the unsharded oracle
product bitwise (and the reference's multiply_parallel partition)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2411_06360_b200 import dist as D


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_matches_reference_workers():
    # kernels.py:222 — bounds = [i * nb // W for i in range(W + 1)]
    for nb in (1, 3, 7, 456, 1490, 5042):
        for W in (1, 2, 3, 4, 8):
            ranges = [D.shard_blocks(nb, W, r) for r in range(W)]
            assert ranges == [(i * nb // W, (i + 1) * nb // W) for i in range(W)]
            assert ranges[0][0] == 0 and ranges[-1][1] == nb
    assert sum(D.slice_lengths(16384, 11, 8)) == 16384
    assert max(D.slice_lengths(65536, 13, 8)) - min(D.slice_lengths(65536, 13, 8)) <= 13


def _worker(rank, world, port, A, v, k, ref, q):
    import torch
    import torch.distributed as dist

    from oracle import c_oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c0, c1 = D.shard_columns(A.shape[1], k, world, rank)
        (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A[:, c0:c1], k)
        local = c_oracle.multiply_parallel(v, pb, nb, c1 - c0, k, True, 1)
        full = D.gather_output(torch.from_numpy(local), A.shape[1], k).numpy()
        q.put((rank, bool(np.array_equal(full, ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,cols,k", [(64, 100, 4), (257, 333, 6), (1024, 1023, 9)])
def test_sharded_multiply_gloo_world2(rows, cols, k):
    from oracle import c_oracle
    rng = np.random.default_rng([rows, cols, k])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    v = rng.integers(-100, 101, size=rows).astype(np.float64)
    (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A, k)
    ref = c_oracle.multiply_parallel(v, pb, nb, cols, k, True, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, A, v, k, ref, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: True, 1: True}
