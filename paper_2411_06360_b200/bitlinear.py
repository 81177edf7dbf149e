"""BitLinear-style decode layer on the RSR++ path.

A fixed ternary weight matrix W [in_features, out_features] (the reference's v · A
orientation: activations are row vectors) is preprocessed once into a device index; every
forward is one `multiply_ternary` (or `multiply_batched` for [B, in] inputs) on the current
stream, and a chain of layers can be captured in one CUDA graph (single vectors never sync;
int32 [B, in] batches run the batch-native kernel, which never syncs once its batch plan —
built on the first batched call — exists, include/rsr_b200.h).  An optional
per-output scale (BitNet's absmean weight scale) is applied after the integer/fixed-point
product.
"""

from __future__ import annotations

import numpy as np

from .core import TernaryMatrix
from .indexer import optimal_k_b200, preprocess_ternary
from .kernels import multiply_batched, multiply_ternary


def _torch():
    import torch
    return torch


class BitLinear(_torch().nn.Module):
    """y = x · W (+ scale) with W ternary [in_features, out_features] held as an RSR index.

    weight: int8 CUDA tensor / NumPy array / TernaryMatrix with entries in {-1, 0, 1}.
    k: block width (default: the B200 tuner, optimal_k_b200(in_features, out_features)).
    scale: optional float or [out_features] tensor multiplied into the output.
    """

    def __init__(self, weight, k: int | None = None, variant: str = "rsrpp", scale=None):
        super().__init__()
        torch = _torch()
        if isinstance(weight, TernaryMatrix):
            rows, cols = weight.entries.shape
        else:
            rows, cols = weight.shape
        self.in_features, self.out_features = int(rows), int(cols)
        self.k = int(k) if k is not None else optimal_k_b200(self.in_features, self.out_features)
        self.variant = variant
        if isinstance(weight, np.ndarray):
            weight = TernaryMatrix(weight.astype(np.int8))
        self.index = preprocess_ternary(weight, self.k)
        if scale is None:
            self.scale = None
        else:
            self.register_buffer("scale", torch.as_tensor(scale, dtype=torch.float32, device="cuda"))

    def forward(self, x):
        torch = _torch()
        if x.dim() == 1:
            y = multiply_ternary(x, self.index, self.variant)
        elif x.dim() == 2:
            y = multiply_batched(x, self.index, self.variant)
        else:
            raise ValueError("BitLinear expects [in_features] or [batch, in_features] inputs")
        if self.scale is not None:
            y = y.to(torch.float32) * self.scale
        return y

    def extra_repr(self) -> str:
        return f"in_features={self.in_features}, out_features={self.out_features}, k={self.k}, variant={self.variant}"


class FusedBitLinear(_torch().nn.Module):
    """Several BitLinear layers that read the same input (q / k / v, or gate / up) as ONE RSR
    index over their concatenated columns [W_1 | W_2 | ...]: one multiply per input instead of
    one per layer, so the fixed per-launch cost (first keys from HBM, the last block's fold) is
    paid once and the blocks of all layers fill the SMs together.  forward returns one output
    per layer (views of the fused result); each equals the separate layer's output bitwise
    (integer activations) — column blocks may straddle two layers, which only changes which
    columns a block holds, never a column's value."""

    def __init__(self, weights, k: int | None = None, variant: str = "rsrpp", scales=None):
        super().__init__()
        torch = _torch()
        mats = []
        for w in weights:
            if isinstance(w, TernaryMatrix):
                w = w.entries
            mats.append(torch.as_tensor(np.asarray(w) if isinstance(w, np.ndarray) else w).to(device="cuda", dtype=torch.int8))
        rows = {int(m.shape[0]) for m in mats}
        if len(rows) != 1:
            raise ValueError("fused layers must share in_features")
        self.in_features = rows.pop()
        self.out_features = [int(m.shape[1]) for m in mats]
        W = torch.cat(mats, dim=1).contiguous()
        self.k = int(k) if k is not None else optimal_k_b200(self.in_features, sum(self.out_features))
        self.variant = variant
        self.index = preprocess_ternary(W, self.k)
        self._splits = list(self.out_features)
        self.scales = None if scales is None else [
            None if sc is None else torch.as_tensor(sc, dtype=torch.float32, device="cuda") for sc in scales]

    def forward(self, x):
        torch = _torch()
        if x.dim() == 1:
            y = multiply_ternary(x, self.index, self.variant)
        elif x.dim() == 2:
            y = multiply_batched(x, self.index, self.variant)
        else:
            raise ValueError("FusedBitLinear expects [in_features] or [batch, in_features] inputs")
        outs = list(torch.split(y, self._splits, dim=-1))
        if self.scales is not None:
            outs = [o if sc is None else o.to(torch.float32) * sc for o, sc in zip(outs, self.scales)]
        return tuple(outs)

    def extra_repr(self) -> str:
        return f"in_features={self.in_features}, out_features={self.out_features}, k={self.k}, variant={self.variant}"


def llama3_8b_mlp_shapes() -> list[tuple[str, int, int]]:
    """The BitNet b1.58 Llama-3-8B layer shapes of BASELINE.json (v · A: [in, out])."""
    return [("q_proj", 4096, 4096), ("o_proj", 4096, 4096), ("gate_proj", 4096, 14336),
            ("up_proj", 4096, 14336), ("down_proj", 14336, 4096)]
