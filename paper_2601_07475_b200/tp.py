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

* SequenceParallelColumnLinear: the Megatron sequence-parallel layout.
  The previous row-parallel layer reduce-scatters its output over tokens (RowParallelLinear
  with reduce="scatter"), so each rank holds M/P rows of the residual stream; the next
  column-parallel layer quantizes only ITS rows (optionally with the fused RMSNorm)
  and all-gathers the packed NVFP4 codes + block scales -- Kp/2 + Kp/16 bytes per row
  instead of 2K for a bf16 all-gather (0.28x at K = 4096) -- then runs its N-shard GEMM over
  all M rows.  The redundant per-rank quantize of the replicated input disappears.  The
  gathered codes are bit-identical to quantizing the full activation (quantization is
  per row), so the outputs equal the column-parallel layer's.

* RowParallelLinear(reduce="fused") (second half): the all-reduce is fused into the
  GEMM epilogue (arc_gemm_reduce): the fp32 output is a torch symmetric-memory buffer mapped on every
  rank; each rank's GEMM adds its partial into every rank's buffer as its tiles finish -- one
  multimem.red per element into the NVLS multicast address when the NVSwitch supports it (the switch
  sums; each rank sends its partial once), else red.add into each peer's buffer over NVLink P2P.
  Symmetric-memory barriers zero-fence the buffers before and publish the sum after.

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


def _all_gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """Every rank's t concatenated along dim 0 in rank order (NCCL all_gather_into_tensor on GPUs)."""
    world = dist.get_world_size(group)
    t = t.contiguous()
    out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if t.is_cuda:
        dist.all_gather_into_tensor(out, t, group=group)
    else:  # gloo
        dist.all_gather(list(out.chunk(world)), t, group=group)
    return out


def _reduce_scatter_rows(y: torch.Tensor, group=None) -> torch.Tensor:
    """Sum over ranks, rank r keeps rows [r M/P, (r+1) M/P) (NCCL reduce_scatter_tensor on GPUs)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m = y.shape[0]
    if m % world:
        raise ValueError(f"M = {m} not divisible by {world} ranks")
    if y.is_cuda:
        out = torch.empty((m // world,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
        dist.reduce_scatter_tensor(out, y.contiguous(), op=dist.ReduceOp.SUM, group=group)
        return out
    y = y.clone()  # gloo has no reduce-scatter: all-reduce, keep this rank's rows
    dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
    return y[rank * (m // world):(rank + 1) * (m // world)].contiguous()


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

    def symmetric_output(self, M: int, device):
        """fp32 [M][N] output buffer shared by every rank (torch symmetric memory) and its handle, cached per M."""
        key = (M, str(device))
        cache = self.__dict__.setdefault("_symm", {})
        if key not in cache:
            if hasattr(self.backend, "symmetric_buffer"):
                cache[key] = self.backend.symmetric_buffer((M, self.qweight_N()), self.group)
            else:
                import torch.distributed._symmetric_memory as symm_mem
                buf = symm_mem.empty((M, self.qweight_N()), dtype=torch.float32, device=device)
                group = self.group if self.group is not None else dist.group.WORLD
                cache[key] = (buf, symm_mem.rendezvous(buf, group))
        return cache[key]

    def qweight_N(self) -> int:
        return int(self.qweight.codes.shape[0])

    def forward(self, x_shard: torch.Tensor, out_dtype=torch.float32, reduce="all") -> torch.Tensor:
        """x_shard: this rank's [M, K/P] slice of the activation.  reduce: "all" (all-reduce, every rank
        gets Y), "fused" (the all-reduce fused into the GEMM epilogue through symmetric memory: NVLS
        multicast or P2P; the returned tensor is the shared buffer, valid until the next fused call),
        "scatter" (reduce-scatter over tokens, rank r gets rows [r M/P, (r+1) M/P): the sequence-parallel
        layout) or None (the partial Y_r)."""
        if reduce == "fused":
            M = x_shard.shape[0]
            buf, h = self.symmetric_output(M, x_shard.device)
            buf.zero_()
            h.barrier()  # every rank's buffer is zero before any rank adds into it
            codes, sf = self.backend.quantize_activation(x_shard, self.profile)
            mc = int(h.multicast_ptr) if getattr(h, "has_multicast_support", False) and h.multicast_ptr else 0
            self.backend.gemm_reduce(codes, sf, self.profile.gs, self.qweight, ldy=self.qweight_N(), mc_ptr=mc,
                                     peer_ptrs=list(h.buffer_ptrs))
            h.barrier()  # every rank's contribution has landed
            return buf if out_dtype == torch.float32 else buf.to(out_dtype)
        y = self.backend.linear(x_shard, self.profile, self.qweight, out_dtype=out_dtype)
        if reduce is True or reduce == "all":
            if self.shard.world > 1 or self.group is not None:
                dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        elif reduce == "scatter":
            y = _reduce_scatter_rows(y, self.group)
        return y


class SequenceParallelColumnLinear:
    """Column-parallel ARC linear fed from M/P token rows per rank: quantize the local rows (optionally
    RMSNorm-fused), all-gather the packed codes + block scales, GEMM over all M rows for this N shard."""

    def __init__(self, weight_full: torch.Tensor, profile, rank: int, world: int, backend=None, group=None):
        self.backend = backend or _default_backend()
        N = weight_full.shape[0]
        lo, hi = shard_range(N, rank, world, align=8)
        self.shard = ShardInfo(rank, world, lo, hi)
        self.group = group
        self.profile = profile
        self.qweight = self.backend.quantize_weight(weight_full[lo:hi].contiguous(), profile)

    def gather_quantized(self, x_rows: torch.Tensor, gamma=None, eps: float = 1e-5):
        """(codes [M][Kp/2], scales) of all ranks' rows: each rank quantizes its M/P rows; the 128x4 scale
        tiles of 128-row blocks concatenate, so M/P must be a multiple of 128."""
        m_loc = x_rows.shape[0]
        if m_loc % 128:
            raise ValueError(f"sequence-parallel rows per rank ({m_loc}) must be a multiple of 128")
        if gamma is not None:
            codes, sf = self.backend.rmsnorm_quantize_activation(x_rows, gamma, eps, self.profile)
        else:
            codes, sf = self.backend.quantize_activation(x_rows, self.profile)
        codes_all = _all_gather_rows(codes, self.group)
        sf_all = _all_gather_rows(sf.reshape(m_loc // 128, -1), self.group).reshape(-1)
        return codes_all, sf_all

    def forward(self, x_rows: torch.Tensor, gamma=None, eps: float = 1e-5, out_dtype=torch.bfloat16):
        codes, sf = self.gather_quantized(x_rows, gamma, eps)
        return self.backend.gemm(codes, sf, self.profile.gs, self.qweight, out_dtype=out_dtype)
