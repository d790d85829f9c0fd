"""CPU stand-in for the libarc.so binding with the interface paper_2601_07475_b200.tp
expects (calibrate / quantize_weight / linear), built on the oracle.  Test-only: it
lets the tensor-parallel host logic run under torch.distributed gloo on CPU."""
from dataclasses import dataclass

import numpy as np
import torch

import oracle


@dataclass
class Prof:
    perm: np.ndarray
    S: int
    gs: float
    layout: int


@dataclass
class QW:
    codes: np.ndarray
    sf: np.ndarray
    gs: float


class OracleBackend:
    def calibrate(self, batches, s_override=-1, layout=0):
        cm = None
        for b in batches:
            cm = oracle.calib_absmax(oracle.as_bf16_bits(b), cm)
        sel = oracle.select_outliers(cm, s_override)
        return Prof(sel["perm"], sel["S"], sel["gs"], layout)

    def quantize_weight(self, w, prof):
        gs_w = oracle.tensor_scale(float(w.float().abs().max()))
        codes, sf = oracle.quantize_weight(oracle.as_bf16_bits(w), prof.perm, prof.S, gs_w, prof.layout)
        return QW(codes, sf, gs_w)

    def linear(self, x, prof, qw, out_dtype=torch.float32):
        ac, asf = oracle.quantize_activation(oracle.as_bf16_bits(x), prof.perm, prof.S, prof.gs, prof.layout)
        y, _ = oracle.gemm_reference(ac, asf, qw.codes, qw.sf, prof.gs, qw.gs)
        return torch.from_numpy(y).to(out_dtype)

    def quantize_activation(self, x, prof):
        ac, asf = oracle.quantize_activation(oracle.as_bf16_bits(x), prof.perm, prof.S, prof.gs, prof.layout)
        return torch.from_numpy(ac), torch.from_numpy(asf)

    def rmsnorm_quantize_activation(self, x, gamma, eps, prof):
        y = oracle.rmsnorm(oracle.as_bf16_bits(x), oracle.as_bf16_bits(gamma), eps)
        ac, asf = oracle.quantize_activation(y, prof.perm, prof.S, prof.gs, prof.layout)
        return torch.from_numpy(ac), torch.from_numpy(asf)

    def gemm(self, codes, sf, gs, qw, out_dtype=torch.float32):
        y, _ = oracle.gemm_reference(codes.numpy(), sf.numpy(), qw.codes, qw.sf, gs, qw.gs)
        return torch.from_numpy(y).to(out_dtype)

    def linear_bound(self, x, prof, qw):
        ac, asf = oracle.quantize_activation(oracle.as_bf16_bits(x), prof.perm, prof.S, prof.gs, prof.layout)
        return oracle.gemm_reference(ac, asf, qw.codes, qw.sf, prof.gs, qw.gs)

    # --- the buffer-level calls bench.py's step makes (bench.Site / bench.run_step) ---
    def buffer_sizes(self, rows, K, S):
        Kp = oracle.kp(K, S)
        return Kp, rows * Kp // 2, oracle.sf_rows_padded(rows) * Kp // 16

    class Workspace:
        def __init__(self, device=None):
            self.device = device

    def quantize_activation_into(self, x, prof, codes, sf):
        ac, asf = oracle.quantize_activation(oracle.as_bf16_bits(x), prof.perm, prof.S, prof.gs, prof.layout)
        codes.copy_(torch.from_numpy(ac))
        sf.copy_(torch.from_numpy(asf.reshape(-1)))
        return codes, sf

    def gemm_into(self, codes, sf, gs, qw, out):
        y, _ = oracle.gemm_reference(codes.numpy(), sf.numpy(), qw.codes, qw.sf, gs, qw.gs)
        out.copy_(torch.from_numpy(y).to(out.dtype))
        return out


class BenchOracleBackend(OracleBackend):
    """OracleBackend with bench.py's in-place call signatures (quantize_activation(x, prof, codes, sf),
    gemm(codes, sf, gs, qw, out=, ws=))."""

    def quantize_activation(self, x, prof, codes=None, sf=None):
        if codes is None:
            return super().quantize_activation(x, prof)
        return self.quantize_activation_into(x, prof, codes, sf)

    def gemm(self, codes, sf, gs, qw, out_dtype=torch.float32, out=None, ws=None):
        if out is None:
            return super().gemm(codes, sf, gs, qw, out_dtype)
        return self.gemm_into(codes, sf, gs, qw, out)


# --- fused row-parallel reduction (tp.RowParallelLinear(reduce="fused")): a CPU emulation of the
# symmetric output buffer and of arc_gemm_reduce, whose every-rank-adds-into-every-buffer semantics
# equals adding the all-reduced partials into each rank's (zeroed) buffer ---
_SYMM_BUFS = {}


class _SymmHandle:
    def __init__(self, buf, group):
        self.group = group
        self.has_multicast_support = False
        self.multicast_ptr = 0
        self.buffer_ptrs = [id(buf)]

    def barrier(self):
        import torch.distributed as dist
        dist.barrier(group=self.group)


def _symmetric_buffer(self, shape, group):
    buf = torch.zeros(shape, dtype=torch.float64)
    _SYMM_BUFS[id(buf)] = buf
    return buf, _SymmHandle(buf, group)


def _gemm_reduce(self, codes, sf, gs, qw, ldy, mc_ptr=0, peer_ptrs=()):
    import torch.distributed as dist
    y, _ = oracle.gemm_reference(codes.numpy(), sf.numpy(), qw.codes, qw.sf, gs, qw.gs)
    t = torch.from_numpy(y)
    dist.all_reduce(t)
    _SYMM_BUFS[peer_ptrs[0]] += t


OracleBackend.symmetric_buffer = _symmetric_buffer
OracleBackend.gemm_reduce = _gemm_reduce
