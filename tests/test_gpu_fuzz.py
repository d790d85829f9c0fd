"""Seeded shape fuzz of the quantize kernels against the oracle (bit-exact): random K (multiples of
16 up to 20000, covering every ring configuration incl. one-row tiles with odd Kp/64), S, M and
layout, activation and weight modes, plus the RMSNorm and SiLU-mul producers on a subset."""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_07475_b200 import synth
from _helpers import dev_bits, valid_sf_mask

pytestmark = pytest.mark.gpu

_rng = np.random.default_rng(2026)
CASES = []
for _ in range(24):
    K = int(_rng.integers(1, 1250)) * 16
    S = int(min(K, int(_rng.integers(0, 33)) * 16))
    M = int(_rng.integers(1, 300))
    CASES.append((M, K, S, int(_rng.integers(0, 2))))


@pytest.mark.parametrize("M,K,S,layout", CASES)
def test_quantize_fuzz(M, K, S, layout):
    from paper_2601_07475_b200 import arc as A
    st = synth.Structure(K, max(min(S, K), 16) if K >= 16 else 1, seed=K + S)
    x = synth.activation(M, K, st, seed=M, device="cuda")
    w = synth.weight(40, K, seed=K, device="cuda")
    prof = A.calibrate([synth.activation(64, K, st, seed=7, device="cuda")], s_override=S, layout=layout)
    codes, sf = A.quantize_activation(x, prof)
    qw = A.quantize_weight(w, prof)
    torch.cuda.synchronize()
    perm, gs = prof.perm.cpu().numpy(), float(prof.gs.item())
    Kp = oracle.kp(K, S)
    ma, mw = valid_sf_mask(M, Kp), valid_sf_mask(40, Kp)
    oc, osf = oracle.quantize_activation(dev_bits(x), perm, S, gs, layout)
    assert np.array_equal(codes.cpu().numpy(), oc)
    assert np.array_equal(sf.cpu().numpy()[ma], osf[ma]), "activation scale bytes differ"
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, S, float(qw.gs.item()), layout)
    assert np.array_equal(qw.codes.cpu().numpy(), bc)
    assert np.array_equal(qw.sf.cpu().numpy()[mw], bsf[mw]), "weight scale bytes differ"
    if K <= 16384 and M <= 64:
        g = synth.rmsnorm_weight(K, seed=3, device="cuda")
        cn, sn = A.rmsnorm_quantize_activation(x, g, 1e-5, prof)
        gu = synth.gate_up(M, K, st, seed=4, device="cuda")
        cs, ss = A.silu_mul_quantize_activation(gu, prof)
        torch.cuda.synchronize()
        on, osn = oracle.quantize_activation(oracle.rmsnorm(dev_bits(x), dev_bits(g), 1e-5), perm, S, gs, layout)
        assert np.array_equal(cn.cpu().numpy(), on)
        assert np.array_equal(sn.cpu().numpy()[ma], osn[ma]), "RMSNorm-quantize scale bytes differ"
        os_, oss = oracle.quantize_activation(oracle.silu_mul(dev_bits(gu)), perm, S, gs, layout)
        assert np.array_equal(cs.cpu().numpy(), os_)
        assert np.array_equal(ss.cpu().numpy()[ma], oss[ma]), "SiLU-mul-quantize scale bytes differ"


_rng2 = np.random.default_rng(7)
GEMM_CASES = []
for _ in range(12):
    K = int(_rng2.integers(1, 160)) * 16
    S = int(min(K, int(_rng2.integers(0, 9)) * 16))
    GEMM_CASES.append((int(_rng2.integers(1, 700)), int(_rng2.integers(1, 300)) * 8, K, S))


@pytest.mark.parametrize("M,N,K,S", GEMM_CASES)
def test_gemm_fuzz(M, N, K, S):
    """Random M (split-K and tile edges), N, K, S: the GEMM within the north_star bound of the
    oracle's exact GEMM, fp32 output."""
    from paper_2601_07475_b200 import arc as A
    st = synth.Structure(K, max(S, 16), seed=N)
    x = synth.activation(M, K, st, seed=M + 1, device="cuda")
    w = synth.weight(N, K, seed=N + 1, device="cuda")
    prof = A.calibrate([synth.activation(64, K, st, seed=9, device="cuda")], s_override=S)
    qw = A.quantize_weight(w, prof)
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                        qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()))
    err = np.abs(y.cpu().numpy().astype(np.float64) - yref)
    assert (err <= bound).all(), f"worst err/bound {np.max(err / np.maximum(bound, 1e-300))}"


@pytest.mark.parametrize("M,N,K,S", [(16, 34, 4096, 128), (7, 130, 2048, 64), (64, 1026, 14336, 128),
                                     (3, 6, 1024, 16)])
def test_gemm_split_k_ragged_n(M, N, K, S):
    """decode-size M takes the split-K path; N not a multiple of 4 must not misalign the
    fp32 partial stores (partial rows are padded to round_up(N, 4)).  fp32 and bf16 outputs."""
    from paper_2601_07475_b200 import arc as A
    st = synth.Structure(K, max(S, 16), seed=N)
    x = synth.activation(M, K, st, seed=M + 11, device="cuda")
    w = synth.weight(N, K, seed=N + 12, device="cuda")
    prof = A.calibrate([synth.activation(64, K, st, seed=13, device="cuda")], s_override=S)
    qw = A.quantize_weight(w, prof)
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    yb = torch.empty(M, (N + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")[:, :N]
    A.gemm(codes, sf, prof.gs, qw, out=yb)
    torch.cuda.synchronize()
    yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                        qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()))
    err = np.abs(y.cpu().numpy().astype(np.float64) - yref)
    assert (err <= bound).all(), f"worst err/bound {np.max(err / np.maximum(bound, 1e-300))}"
    assert torch.equal(yb, y.to(torch.bfloat16))
