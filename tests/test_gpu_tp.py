"""Tensor-parallel wrappers on the GPU with the real libarc.so backend and an NCCL
process group (world size 1 on the single test GPU): the row-parallel layer runs its
NCCL all-reduce path; both layers match the oracle (per-shard, north_star tolerance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
from paper_2601_07475_b200 import synth
from _helpers import dev_bits

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_tp_layers_world1_nccl(pg):
    from paper_2601_07475_b200 import arc, tp
    M, K, N = 64, 1024, 512
    st = synth.Structure(K, 32, seed=0)
    x = synth.activation(M, K, st, seed=1, device="cuda")
    cal = synth.activation(512, K, st, seed=1000, device="cuda")
    w = synth.weight(N, K, seed=2, device="cuda")
    prof = arc.calibrate([cal])
    col = tp.ColumnParallelLinear(w, prof, 0, 1)
    row = tp.RowParallelLinear(w, cal, 0, 1, group=pg)
    y_col = col.forward(x, out_dtype=torch.float32)
    y_row = row.forward(x, out_dtype=torch.float32)
    torch.cuda.synchronize()
    for lin, y in ((col, y_col), (row, y_row)):
        p = lin.profile
        perm, gs, gs_w = p.perm.cpu().numpy(), float(p.gs.item()), float(lin.qweight.gs.item())
        ac, asf = oracle.quantize_activation(dev_bits(x), perm, p.S, gs)
        bc, bsf = oracle.quantize_weight(dev_bits(w), perm, p.S, gs_w)
        yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
        assert np.all(np.abs(y.cpu().numpy().astype(np.float64) - yref) <= bound)


def test_sequence_parallel_world1_nccl(pg):
    """SURVEY f2 path on the GPU (NCCL all_gather_into_tensor / reduce_scatter_tensor at world 1):
    the gathered codes and scales equal the direct quantization, the SP column output equals
    arc.gemm on them, the RMSNorm-fused variant equals arc.linear_rmsnorm."""
    from paper_2601_07475_b200 import arc, tp
    M, K, N = 256, 1024, 512
    st = synth.Structure(K, 32, seed=3)
    x = synth.activation(M, K, st, seed=4, device="cuda")
    cal = synth.activation(512, K, st, seed=1001, device="cuda")
    w = synth.weight(N, K, seed=5, device="cuda")
    gamma = synth.rmsnorm_weight(K, seed=6, device="cuda")
    prof = arc.calibrate([cal])
    sp = tp.SequenceParallelColumnLinear(w, prof, 0, 1, group=pg)
    codes, sf = sp.gather_quantized(x)
    c0, s0 = arc.quantize_activation(x, prof)
    y = sp.forward(x, out_dtype=torch.float32)
    y0 = arc.gemm(c0, s0, prof.gs, sp.qweight, out_dtype=torch.float32)
    yn = sp.forward(x, gamma=gamma, eps=1e-5, out_dtype=torch.float32)
    yn0 = arc.linear_rmsnorm(x, gamma, 1e-5, prof, sp.qweight, out_dtype=torch.float32)
    row = tp.RowParallelLinear(w, cal, 0, 1, group=pg)
    y_all = row.forward(x, out_dtype=torch.float32, reduce="all")
    y_sc = row.forward(x, out_dtype=torch.float32, reduce="scatter")
    torch.cuda.synchronize()
    assert torch.equal(codes, c0) and torch.equal(sf, s0)
    assert torch.equal(y, y0) and torch.equal(yn, yn0)
    assert torch.equal(y_sc, y_all)


@pytest.mark.parametrize("M,K,N", [(256, 2048, 512), (16, 4096, 1024), (300, 1024, 130)])
def test_gemm_reduce_peers_equals_gemm(M, K, N):
    """arc_gemm_reduce in P2P mode with this GPU as the only peer: zero + partial == the plain fp32 GEMM
    (prefill epilogue and split-K reduce-kernel paths; ragged N uses the scalar reductions)."""
    from paper_2601_07475_b200 import arc
    st = synth.Structure(K, 32, seed=M)
    x = synth.activation(M, K, st, seed=M + 1, device="cuda")
    w = synth.weight(N, K, seed=N, device="cuda")
    prof = arc.calibrate([synth.activation(256, K, st, seed=5, device="cuda")], s_override=32)
    qw = arc.quantize_weight(w, prof)
    codes, sf = arc.quantize_activation(x, prof)
    y = arc.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    ldy = (N + 3) // 4 * 4
    out = torch.zeros(M, ldy, dtype=torch.float32, device="cuda")
    arc.gemm_reduce(codes, sf, prof.gs, qw, ldy=ldy, peer_ptrs=[out.data_ptr()])
    torch.cuda.synchronize()
    if M > 64:
        assert torch.equal(out[:, :N], y)
    else:
        # decode-size M: arc_gemm runs the cluster split-K kernel (partials summed in DSMEM, then scaled),
        # arc_gemm_reduce the split-K kernel + reduce kernel (scaled partials summed): same math, another
        # fp32 summation order -- both within 1e-5 * sum|ab| of the exact GEMM (test_gpu_decode_cluster)
        assert torch.allclose(out[:, :N], y, rtol=1e-5, atol=1e-6 * float(y.abs().max()))
    p1 = out[:, :N].clone()
    arc.gemm_reduce(codes, sf, prof.gs, qw, ldy=ldy, peer_ptrs=[out.data_ptr(), out.data_ptr()])
    torch.cuda.synchronize()
    assert torch.allclose(out[:, :N], 3 * p1, rtol=1e-6, atol=0)  # every peer receives each partial


def test_row_parallel_fused_reduce_world1_nccl(pg):
    """tp.RowParallelLinear(reduce="fused") over torch symmetric memory (NVLS multicast when the box has
    it, else P2P) equals the NCCL all-reduce path at world size 1, and the multicast mode itself (when
    available) adds exactly once."""
    from paper_2601_07475_b200 import arc, tp
    import torch.distributed._symmetric_memory as symm_mem
    M, K, N = 256, 2048, 512
    st = synth.Structure(K, 32, seed=3)
    x = synth.activation(M, K, st, seed=4, device="cuda")
    cal = synth.activation(256, K, st, seed=5, device="cuda")
    w = synth.weight(N, K, seed=6, device="cuda")
    row = tp.RowParallelLinear(w, cal, 0, 1, backend=arc)
    y_ar = row.forward(x, out_dtype=torch.float32, reduce="all").clone()
    y_f1 = row.forward(x, reduce="fused").clone()
    y_f2 = row.forward(x, reduce="fused").clone()
    torch.cuda.synchronize()
    assert torch.equal(y_f1, y_ar) and torch.equal(y_f2, y_ar)
    buf, h = row.symmetric_output(M, x.device)
    print("multicast support:", bool(getattr(h, "has_multicast_support", False)), "multicast_ptr:", h.multicast_ptr)
    if getattr(h, "has_multicast_support", False) and h.multicast_ptr:
        codes, sf = arc.quantize_activation(x, row.profile)
        buf.zero_()
        arc.gemm_reduce(codes, sf, row.profile.gs, row.qweight, ldy=N, mc_ptr=int(h.multicast_ptr))
        torch.cuda.synchronize()
        assert torch.equal(buf, y_ar)
