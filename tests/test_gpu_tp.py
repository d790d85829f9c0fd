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
