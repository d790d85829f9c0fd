"""Tensor-parallel ARC linear layers over torch.distributed (BASELINE.json north_star:
"column-parallel over N with no communication, and row-parallel over the extended K
with an NCCL all-reduce over NVLink").

The paper is single-GPU; this is the build's own sharding of the
ARC linear:

* ColumnParallelLinear: weight rows (output features N) split into P contiguous
  shards.  The activation is replicated, so every rank uses the SAME calibration
  profile (perm, S, gs_x) and computes Y[:, shard r] with one arc_linear.  No
  communication; the output stays sharded over N.
* RowParallelLinear: input features K split into P contiguous slices, as a
  preceding column-parallel layer leaves them.  Each rank calibrates ITS slice
  (perm_r, S_r, gs_r: the outlier channels of that slice), quantizes W[:, slice r]
  with perm_r (outlier columns duplicated), computes the partial
  Y_r = X_r W_r^T over K/P + S_r, and the partials are summed with one all-reduce
  (NCCL over NVLink/NVSwitch on GPUs).  Per-rank block groupings differ from the
  unsharded layer, so the result equals sum_r linear_r, not the 1-GPU layer.

The compute backend is the ctypes binding of libarc.so by default; tests inject a
CPU backend to exercise this host logic with the gloo backend on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int, align: int = 16):
    """Contiguous [lo, hi) shard of `total` for `rank`; shard sizes are multiples of
    `align` (the NVFP4 block, so K shards keep K % 16 == 0)."""
    if total % (align * world):
        raise ValueError(f"{total} not divisible into {world} shards of multiples of {align}")
    step = total // world
    return rank * step, (rank + 1) * step


def _default_backend():
    from paper_2601_07475_b200 import arc  # fails loudly if libarc.so is missing
    return arc


@dataclass
class ShardInfo:
    rank: int
    world: int
    lo: int
    hi: int


class ColumnParallelLinear:
    """Y[:, N-shard] = ARC-linear(X, W[N-shard, :]) with a replicated input and profile."""

    def __init__(self, weight_full: torch.Tensor, profile, rank: int, world: int, backend=None):
        self.backend = backend or _default_backend()
        N = weight_full.shape[0]
        lo, hi = shard_range(N, rank, world, align=8)
        self.shard = ShardInfo(rank, world, lo, hi)
        self.profile = profile
        self.qweight = self.backend.quantize_weight(weight_full[lo:hi].contiguous(), profile)

    def forward(self, x: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
        return self.backend.linear(x, self.profile, self.qweight, out_dtype=out_dtype)


class RowParallelLinear:
    """Y = all_reduce_r ARC-linear(X[:, K-slice r], W[:, K-slice r]) with per-rank calibration."""

    def __init__(self, weight_full: torch.Tensor, calib_full: torch.Tensor, rank: int, world: int,
                 s_override: int = -1, backend=None, group=None, layout: int = 0):
        self.backend = backend or _default_backend()
        K = weight_full.shape[1]
        lo, hi = shard_range(K, rank, world, align=16)
        self.shard = ShardInfo(rank, world, lo, hi)
        self.group = group
        # per-rank calibration on the rank's input slice (its outlier channels)
        self.profile = self.backend.calibrate([calib_full[:, lo:hi].contiguous()], s_override=s_override,
                                              layout=layout)
        self.qweight = self.backend.quantize_weight(weight_full[:, lo:hi].contiguous(), self.profile)

    def forward(self, x_shard: torch.Tensor, out_dtype=torch.float32, reduce: bool = True) -> torch.Tensor:
        """x_shard: this rank's [M, K/P] slice of the activation."""
        y = self.backend.linear(x_shard, self.profile, self.qweight, out_dtype=out_dtype)
        if reduce and self.shard.world > 1:
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y
