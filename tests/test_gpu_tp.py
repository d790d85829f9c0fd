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
