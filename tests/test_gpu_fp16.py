"""GPU parity of the fp16 input path (SURVEY 8(b) arc_dtype_t ARC_FP16; arc.h *_ex entry points): fp16 rows are
decoded exactly to fp32 and go through the same STAGE arithmetic, so codes and scale bytes
are bit-exact against the oracle's fp16 path -- the ring kernel (M > 64) and the decode-size direct-gather
kernel (M <= 64), both layouts, weights; calibration abs-max and the tensor scale equal the oracle's; the fp16
linear is within the GEMM tolerance of the oracle's exact GEMM."""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_07475_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2601_07475_b200 import arc
    assert arc.device_supported()
    return arc


def _f16_bits(t):
    return oracle.as_fp16_bits(t.cpu())


def _sf_equal(got, want, rows, Kp):
    for m in range(rows):
        for c in range(Kp // 16):
            o = oracle.sf_offset(m, c, Kp)
            assert got[o] == want[o], f"scale byte (row {m}, block {c})"


@pytest.mark.parametrize("M,K,S", [(1, 256, 16), (16, 4096, 128), (64, 1024, 64), (200, 4096, 128), (300, 14336, 128),
                                   (130, 512, 0)])
@pytest.mark.parametrize("layout", [0, 1])
def test_fp16_activation_bit_exact(A, M, K, S, layout):
    st = synth.Structure(K, max(S, 16), seed=K + M)
    x = synth.activation(M, K, st, seed=M + 1, device="cuda").to(torch.float16)
    prof = A.calibrate([synth.activation(256, K, st, seed=2, device="cuda").to(torch.float16)], s_override=S,
                       layout=layout)
    c, sf = A.quantize_activation(x, prof)
    torch.cuda.synchronize()
    oc, osf = oracle.quantize_activation(_f16_bits(x), prof.perm.cpu().numpy(), prof.S, float(prof.gs.item()), layout,
                                         fp16=True)
    assert np.array_equal(c.cpu().numpy(), oc)
    _sf_equal(sf.cpu().numpy(), osf, M, oracle.kp(K, S))


@pytest.mark.parametrize("N,K,S", [(256, 256, 16), (640, 4096, 128)])
def test_fp16_weight_bit_exact(A, N, K, S):
    st = synth.Structure(K, max(S, 16), seed=N)
    w = synth.weight(N, K, seed=N + 1, device="cuda").to(torch.float16)
    prof = A.calibrate([synth.activation(256, K, st, seed=3, device="cuda")], s_override=S)
    qw = A.quantize_weight(w, prof)
    torch.cuda.synchronize()
    gs_w = float(qw.gs.item())
    assert np.float32(gs_w) == np.float32(oracle.tensor_scale(float(w.float().abs().max().item())))
    bc, bsf = oracle.quantize_weight(_f16_bits(w), prof.perm.cpu().numpy(), prof.S, gs_w, fp16=True)
    assert np.array_equal(qw.codes.cpu().numpy(), bc)
    _sf_equal(qw.sf.cpu().numpy(), bsf, N, oracle.kp(K, S))


def test_fp16_calibration_equals_oracle(A):
    K = 1024
    st = synth.Structure(K, 32, seed=5)
    x = synth.activation(777, K, st, seed=6, device="cuda").to(torch.float16)
    cm = A.calib_absmax(x)
    torch.cuda.synchronize()
    assert np.array_equal(cm.cpu().numpy(), oracle.calib_absmax(_f16_bits(x), fp16=True))


@pytest.mark.parametrize("M", [4, 16, 512])
def test_fp16_linear_vs_oracle(A, M):
    N, K, S = 768, 2048, 64
    st = synth.Structure(K, S, seed=M)
    x = synth.activation(M, K, st, seed=M + 9, device="cuda").to(torch.float16)
    w = synth.weight(N, K, seed=10, device="cuda").to(torch.float16)
    prof = A.calibrate([synth.activation(256, K, st, seed=11, device="cuda").to(torch.float16)], s_override=S)
    qw = A.quantize_weight(w, prof)
    y = A.linear(x, prof, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = sorted({0, M // 2, M - 1})
    perm, gs, gs_w = prof.perm.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item())
    ac, asf = oracle.quantize_activation(_f16_bits(x[torch.as_tensor(rows, device="cuda")]), perm, prof.S, gs,
                                         fp16=True)
    bc, bsf = oracle.quantize_weight(_f16_bits(w), perm, prof.S, gs_w, fp16=True)
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
    err = np.abs(y[rows].cpu().numpy().astype(np.float64) - yref)
    assert (err <= bound).all(), f"worst err/bound {np.max(err / bound)}"
