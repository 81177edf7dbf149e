"""Multi-GPU column-block sharding.

Column blocks are independent, so rank g of G owns the block range
[g*NB//G, (g+1)*NB//G) — the same partition `multiply_parallel` gives its workers
(kernels.py:222) — holds only that shard's index, multiplies it into its disjoint
output slice, and one all-gather (NCCL over NVLink on GPUs; gloo in the CPU tests)
replicates the full output vector.  Slices differ by at most one block, so they are
padded to the largest slice for `all_gather_into_tensor` and compacted afterwards.
"""

from __future__ import annotations

import ctypes

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


class FusedAllGather:
    """Multiply + all-gather in ONE kernel per rank (csrc/multiply.cu, the Gather epilogue of
    rsr_multiply_allgather): as soon as a block is folded its int32 column values are stored into
    every rank's gathered vector over peer memory (NVLink P2P stores overlapping the remaining
    blocks' reductions), and the launch's last CTA signals every rank; `rsr_allgather_wait`
    orders this rank's stream after every rank's slice has landed.  Replaces the
    multiply_sharded launch + NCCL all-gather for single-split shards (rows <= 16384).

    Buffers alternate by call parity: a rank writes call c + 1 into a peer's parity only after
    its own wait for call c, i.e. after every peer launched call c — which each peer's stream
    orders after its use of call c - 1's vector (same parity).  Correct by construction, no
    host synchronisation.

    `peers` gives, per rank, the device pointers of its two gathered buffers and its 64-bit
    signal word; `FusedAllGather.symmetric` builds them from a torch symmetric-memory rendezvous
    (multi-GPU); tests pass local buffers ("virtual ranks" on one GPU)."""

    def __init__(self, local_idx, cols: int, world: int, rank: int, out_ptrs, sig_ptrs, gathered, done,
                 variant: str = "rsrpp"):
        from . import _native
        from .kernels import _use_fold
        lens = slice_lengths(cols, local_idx.k, world)
        if local_idx.cols != lens[rank]:
            raise ValueError(f"local index has {local_idx.cols} columns, the partition gives this rank {lens[rank]}")
        if not 1 <= world <= 8:
            raise ValueError("the fused all-gather handles 1 to 8 ranks")
        self.idx, self.cols, self.world, self.rank = local_idx, cols, world, rank
        self.lens, self.pad = lens, max(lens)
        self.gathered, self.done = gathered, done  # [2][world * pad] int32 (this rank's), local u64 counter
        P = ctypes.c_void_p * 8
        self._outs = [P(*[o[par] for o in out_ptrs] + [None] * (8 - world)) for par in (0, 1)]
        self._sigs = P(*list(sig_ptrs) + [None] * (8 - world))
        self._my_sig = sig_ptrs[rank]
        self.variant = _native.VARIANT_RSRPP if _use_fold(variant) else _native.VARIANT_RSR
        self.calls = 0

    def launch(self, v, local_out=None):
        """Enqueue this rank's multiply + peer stores for the next call (v: CUDA int32 [rows])."""
        import torch
        from . import _native
        if v.dtype != torch.int32 or not v.is_cuda:
            raise ValueError("the fused all-gather multiplies int32 CUDA vectors")
        if v.numel() != self.idx.rows:
            raise ValueError(f"vector length {v.numel()} does not match {self.idx.rows} rows")
        par = self.calls & 1
        self.calls += 1
        if local_out is None:
            local_out = torch.empty(self.idx.cols, dtype=torch.int32, device=v.device)
        _native.check(_native.lib().rsr_multiply_allgather(
            ctypes.byref(self.idx.desc), v.data_ptr(), local_out.data_ptr(), self.variant, self._outs[par], self._sigs,
            self.world, self.rank * self.pad, self.done.data_ptr(), torch.cuda.current_stream().cuda_stream))
        return local_out

    def wait(self):
        """Enqueue the wait for every rank's slice of the last launched call; returns the [cols]
        gathered int32 result (a view of that call's buffer parity when no padding is needed)."""
        import torch
        from . import _native
        _native.check(_native.lib().rsr_allgather_wait(self._my_sig, self.calls * self.world,
                                                       torch.cuda.current_stream().cuda_stream))
        g = self.gathered[(self.calls - 1) & 1]
        if all(n == self.pad for n in self.lens):
            return g[: self.cols]
        return torch.cat([g[r * self.pad: r * self.pad + self.lens[r]] for r in range(self.world)])

    def __call__(self, v, local_out=None):
        """v (CUDA int32, this rank's full input) times the sharded matrix, gathered on every rank."""
        self.launch(v, local_out)
        return self.wait()

    @classmethod
    def symmetric(cls, local_idx, cols: int, group=None, variant: str = "rsrpp"):
        """Peer buffers from torch symmetric memory (NVLink-mapped on multi-GPU nodes)."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        pad = max(slice_lengths(cols, local_idx.k, world))
        dev = torch.device("cuda", torch.cuda.current_device())
        gathered = symm_mem.empty(2 * world * pad, dtype=torch.int32, device=dev).view(2, world * pad)
        sig = symm_mem.empty(1, dtype=torch.int64, device=dev)
        sig.zero_()
        gname = (group or dist.group.WORLD).group_name
        hg = symm_mem.rendezvous(gathered, gname)
        hs = symm_mem.rendezvous(sig, gname)
        dist.barrier(group)
        row = 4 * world * pad  # bytes of one parity
        out_ptrs = [(hg.buffer_ptrs[r], hg.buffer_ptrs[r] + row) for r in range(world)]
        done = torch.zeros(1, dtype=torch.int64, device=dev)
        obj = cls(local_idx, cols, world, rank, out_ptrs, list(hs.buffer_ptrs), gathered, done, variant)
        obj._keep = (hg, hs, sig)
        return obj
