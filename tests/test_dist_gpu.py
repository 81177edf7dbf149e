"""The sharded GPU path itself at world size 2: two processes share cuda:0
(this pool has one GPU per box), each builds ITS column shard's index on the GPU
(dist.preprocess_ternary_shard), multiplies on the GPU and all-gathers over gloo (CPU copies;
the ranks never wait on each other inside a kernel).  The gathered vector must be bitwise
equal to the unsharded multiply_ternary and to the reference partition's result
(multiply_parallel, W = world, kernels.py:209-239)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, A, v, k, q):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2411_06360_b200 as rsr
    from paper_2411_06360_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local_idx = D.preprocess_ternary_shard(A, k, world, rank)
        outs = {}
        for dt in (torch.int32, torch.int64, torch.float64):
            dv = torch.from_numpy(v).to(dt).cuda()
            for variant in ("rsrpp", "rsr"):
                full = D.multiply_sharded(dv, local_idx, A.shape[1], variant=variant)
                assert full.is_cuda and full.dtype == dt
                outs[(str(dt), variant)] = full.double().cpu().numpy()
        c0, c1 = D.shard_columns(A.shape[1], k, world, rank)
        q.put((rank, outs, (c0, c1), local_idx.cols))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,k", [(257, 333, 6), (2048, 1001, 9), (16384, 2050, 11)])
def test_sharded_multiply_world2_on_gpu(rsr, cuda, rows, cols, k):
    from oracle import c_oracle
    rng = np.random.default_rng([rows, cols, k, 2])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    v = rng.integers(-100, 101, size=rows).astype(np.int64)
    (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A, k)
    ref = {var: c_oracle.multiply_parallel(v.astype(np.float64), pb, nb, cols, k, var == "rsrpp", 2)
           for var in ("rsrpp", "rsr")}
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    unsharded = rsr.multiply_ternary(v, idx)
    assert np.array_equal(unsharded, ref["rsrpp"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, A, v, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(2):
        rank, outs, cr, lcols = q.get(timeout=300)
        results[rank] = (outs, cr, lcols)
    for p in procs:
        p.join(timeout=60)
    for rank, (outs, cr, lcols) in results.items():
        assert not isinstance(outs, str), outs
        assert cr[1] - cr[0] == lcols
        for (dt, variant), got in outs.items():
            assert np.array_equal(got, ref[variant]), (rank, dt, variant)
    # the two shards cover the columns exactly, split on a block boundary (kernels.py:222)
    assert results[0][1][0] == 0 and results[0][1][1] == results[1][1][0] and results[1][1][1] == cols
    assert results[0][1][1] % k == 0


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,k,world", [(4096, 1000, 10, 3), (16384, 2050, 11, 4), (300, 77, 6, 8), (1000, 55, 7, 1)])
def test_fused_allgather_virtual_ranks(rsr, cuda, rows, cols, k, world):
    """The fused multiply + all-gather kernel (csrc/multiply.cu Gather epilogue) with `world`
    virtual ranks on one GPU: each rank owns its shard index, its two gathered buffers and its
    signal word; every rank's launch stores its folded columns into ALL ranks' buffers and signals
    them.  All launches of a call are enqueued before any wait (no kernel waits on a kernel that
    is not already queued ahead of it), then each rank's wait + check: every rank's gathered
    vector equals the unsharded product bitwise, over several calls (both buffer parities)."""
    import torch
    from oracle import c_oracle
    from paper_2411_06360_b200 import dist as D
    rng = np.random.default_rng([rows, cols, world])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idxs = [D.preprocess_ternary_shard(A, k, world, r) for r in range(world)]
    pad = max(D.slice_lengths(cols, k, world))
    gathered = [torch.full((2, world * pad), -7, dtype=torch.int32, device="cuda") for _ in range(world)]
    sigs = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
    dones = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
    out_ptrs = [(g[0].data_ptr(), g[1].data_ptr()) for g in gathered]
    sig_ptrs = [s.data_ptr() for s in sigs]
    fags = [D.FusedAllGather(idxs[r], cols, world, r, out_ptrs, sig_ptrs, gathered[r], dones[r],
                             variant="rsrpp" if r % 2 == 0 else "rsr") for r in range(world)]
    for call in range(5):
        v = rng.integers(-100, 101, size=rows).astype(np.int32)
        ref = c_oracle.naive_ternary(v.astype(np.float64), A).astype(np.int64)
        dv = torch.from_numpy(v).cuda()
        locals_ = [f.launch(dv) for f in fags]
        for r, f in enumerate(fags):
            got = f.wait()
            assert np.array_equal(got.cpu().numpy().astype(np.int64), ref), (call, r)
            c0, c1 = D.shard_columns(cols, k, world, r)
            assert np.array_equal(locals_[r].cpu().numpy().astype(np.int64), ref[c0:c1]), (call, r)
        torch.cuda.synchronize()
        assert all(int(s.item()) == (call + 1) * world for s in sigs)


@pytest.mark.gpu
def test_fused_allgather_symmetric_world1(rsr, cuda):
    """The torch symmetric-memory rendezvous path (the multi-GPU plumbing) at world size 1."""
    import torch
    import torch.distributed as dist
    from oracle import c_oracle
    from paper_2411_06360_b200 import dist as D
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except ImportError:  # pragma: no cover
        pytest.skip("torch symmetric memory unavailable")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(3)
        A = rng.integers(-1, 2, size=(2048, 700), dtype=np.int8)
        idx = D.preprocess_ternary_shard(A, 9, 1, 0)
        try:
            fag = D.FusedAllGather.symmetric(idx, 700)
        except Exception as e:  # pragma: no cover - symmetric memory not supported on this box
            pytest.skip(f"symmetric memory rendezvous failed: {e!r}"[:200])
        for _ in range(3):
            v = rng.integers(-100, 101, size=2048).astype(np.int32)
            got = fag(torch.from_numpy(v).cuda())
            assert np.array_equal(got.cpu().numpy().astype(np.int64),
                                  c_oracle.naive_ternary(v.astype(np.float64), A).astype(np.int64))
    finally:
        dist.destroy_process_group()
