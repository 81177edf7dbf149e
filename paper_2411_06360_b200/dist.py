"""Multi-GPU column-block sharding.

Column blocks are independent, so rank g of G owns the block range
[g*NB//G, (g+1)*NB//G) — the same partition `multiply_parallel` gives its workers
(kernels.py:222) — holds only that shard's index, multiplies it into its disjoint
output slice, and one all-gather (NCCL over NVLink on GPUs; gloo in the CPU tests)
replicates the full output vector.  Slices differ by at most one block, so they are
padded to the largest slice for `all_gather_into_tensor` and compacted afterwards.
"""

from __future__ import annotations

import numpy as np


def shard_blocks(nblocks: int, world: int, rank: int) -> tuple[int, int]:
    """Block range of `rank` (kernels.py:222: bounds = [i*nb//W for i in range(W+1)])."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    return rank * nblocks // world, (rank + 1) * nblocks // world


def shard_columns(cols: int, k: int, world: int, rank: int) -> tuple[int, int]:
    """Column range [c0, c1) covered by the rank's blocks."""
    nb = -(-cols // k)
    b0, b1 = shard_blocks(nb, world, rank)
    return min(cols, b0 * k), min(cols, b1 * k)


def slice_lengths(cols: int, k: int, world: int) -> list[int]:
    return [c1 - c0 for c0, c1 in (shard_columns(cols, k, world, r) for r in range(world))]


def gather_output(local_out, cols: int, k: int, group=None):
    """All-gather the ranks' output slices into the full [cols] vector.  NCCL gathers CUDA
    tensors in place (NVLink); a gloo group (CPU tests, or ranks sharing one GPU) gathers
    CPU copies and the result comes back on local_out's device."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    lens = slice_lengths(cols, k, world)
    pad = max(lens)
    if local_out.numel() != lens[dist.get_rank(group)]:
        raise ValueError(f"local slice has {local_out.numel()} columns, the partition gives this rank "
                         f"{lens[dist.get_rank(group)]}")
    dev = local_out.device
    comm_dev = torch.device("cpu") if dist.get_backend(group) == "gloo" else dev
    send = torch.zeros(pad, dtype=local_out.dtype, device=comm_dev)
    send[: local_out.numel()] = local_out.to(comm_dev)
    recv = torch.empty(world * pad, dtype=local_out.dtype, device=comm_dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    parts = [recv[r * pad: r * pad + lens[r]] for r in range(world)]
    return torch.cat(parts).to(dev)


def preprocess_ternary_shard(A, k: int, world: int, rank: int):
    """Index of this rank's column shard of A (host TernaryMatrix / int8 array / CUDA
    tensor [rows, cols]).  The shard starts on a block boundary, so its blocks are exactly
    the global blocks [b0, b1)."""
    import torch

    from .core import TernaryMatrix
    from .indexer import preprocess_ternary
    entries = A.entries if isinstance(A, TernaryMatrix) else A
    cols = entries.shape[1]
    c0, c1 = shard_columns(cols, k, world, rank)
    if isinstance(entries, torch.Tensor):
        shard = entries[:, c0:c1].contiguous()
        if not shard.is_cuda:
            shard = shard.cuda()
    else:
        shard = torch.from_numpy(np.ascontiguousarray(np.asarray(entries, np.int8)[:, c0:c1])).cuda()
    return preprocess_ternary(shard, k)


def multiply_sharded(v, local_idx, cols: int, group=None, variant: str = "rsrpp"):
    """v (CUDA tensor, full length rows) times the sharded matrix: local multiply of this
    rank's blocks (one launch, its disjoint output slice), then all-gather of the slices.
    Returns the full [cols] tensor on v's device; bitwise equal to the unsharded
    multiply_ternary / multiply_rsr and to the reference's multiply_parallel(W=world)."""
    from .indexer import TernaryIndex
    from .kernels import multiply_rsr, multiply_ternary
    mult = multiply_ternary if isinstance(local_idx, TernaryIndex) else multiply_rsr
    local = mult(v, local_idx, variant)
    return gather_output(local, cols, local_idx.k, group)
