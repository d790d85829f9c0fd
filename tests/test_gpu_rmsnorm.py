"""GPU parity of the RMSNorm stage of the fused quantization kernel (Fig.8b
P:397; reduction order and roundings = DESIGN.md reading Q23):

* arc_rmsnorm is bit-exact against the oracle's RMSNorm;
* arc_rmsnorm_quantize_activation (RMSNorm + reorder + primary + residual NVFP4 in one pass)
  is bit-exact against the oracle's quantize_activation of the oracle's RMSNorm (codes and
  the scales of every valid row), in both layouts, across the kernel's ring configurations
  (R = 4 / 2 / 1 rows per tile, 28 primary warps, the two-blocks-per-lane fallback);
* arc_linear_rmsnorm is within the GEMM tolerance of the oracle's exact GEMM."""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_07475_b200 import synth
from _helpers import dev_bits, valid_sf_mask

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2601_07475_b200 import arc
    assert arc.device_supported()
    return arc


def _inputs(M, K, S, seed):
    st = synth.Structure(K, max(S, 16), seed=seed)
    h = synth.activation(M, K, st, seed=seed + 1, device="cuda")
    g = synth.rmsnorm_weight(K, seed=seed, device="cuda")
    return st, h, g


@pytest.mark.parametrize("M,K", [(1, 16), (7, 48), (64, 256), (129, 4096), (33, 4112), (20, 14336), (5, 32768)])
@pytest.mark.parametrize("eps", [1e-5, 0.0])
def test_rmsnorm_bit_exact(A, M, K, eps):
    st, h, g = _inputs(M, K, 16, seed=K + M)
    y = A.rmsnorm(h, g, eps)
    torch.cuda.synchronize()
    ref = oracle.rmsnorm(dev_bits(h), dev_bits(g), eps)
    assert np.array_equal(dev_bits(y), ref)


def test_rmsnorm_strided_rows(A):
    M, K = 40, 1024
    st, h, g = _inputs(M, K + 64, 16, seed=3)
    hv = h[:, :K]  # row stride K + 64
    y = torch.empty(M, K + 128, dtype=torch.bfloat16, device="cuda")[:, :K]
    A.rmsnorm(hv, g[:K].contiguous(), 1e-5, out=y)
    torch.cuda.synchronize()
    assert np.array_equal(dev_bits(y), oracle.rmsnorm(dev_bits(hv), dev_bits(g[:K]), 1e-5))


# K = 4096 (R = 4 ring, 8 primary warps), 14336 (R = 2, 28 primary warps + 2 norm warps = 1024
# threads), 14336 with S = 512 (two residual warps -> the two-blocks-per-lane fallback, R = 1),
# 16384 (two blocks per lane), small / ragged cases
@pytest.mark.parametrize("M,K,S", [(16, 256, 16), (300, 4096, 128), (77, 14336, 128), (9, 14336, 512),
                                   (12, 16384, 256), (130, 1024, 0), (5, 112, 48)])
@pytest.mark.parametrize("layout", [0, 1])
def test_rmsnorm_quantize_bit_exact(A, M, K, S, layout):
    st, h, g = _inputs(M, K, S, seed=M * 3 + K + layout)
    eps = 1e-5
    cal = A.rmsnorm(synth.activation(256, K, st, seed=99, device="cuda"), g, eps)
    prof = A.calibrate([cal], s_override=S, layout=layout)
    codes, sf = A.rmsnorm_quantize_activation(h, g, eps, prof)
    # the unfused chain on the GPU: bit-identical by construction of the shared device code
    c2, s2 = A.quantize_activation(A.rmsnorm(h, g, eps), prof)
    torch.cuda.synchronize()
    y_or = oracle.rmsnorm(dev_bits(h), dev_bits(g), eps)
    oc, osf = oracle.quantize_activation(y_or, prof.perm.cpu().numpy(), S, float(prof.gs.item()), layout)
    mask = valid_sf_mask(M, prof_kp(K, S))
    assert np.array_equal(codes.cpu().numpy(), oc), "fused RMSNorm+quantize codes differ from the oracle"
    assert np.array_equal(sf.cpu().numpy()[mask], osf[mask]), "fused RMSNorm+quantize scales differ"
    assert torch.equal(codes, c2) and torch.equal(sf.view(-1)[torch.from_numpy(mask).cuda()],
                                                  s2.view(-1)[torch.from_numpy(mask).cuda()])


def prof_kp(K, S):
    return (K + S + 63) // 64 * 64


def test_rmsnorm_quantize_full_size_sampled_rows(A):
    """The bench's attention-input site at full prefill size (M = 8192, K = 4096, S = 128),
    bit-exact on sampled rows (the oracle runs row by row)."""
    M, K, S = 8192, 4096, 128
    st, h, g = _inputs(M, K, S, seed=11)
    prof = A.calibrate([A.rmsnorm(synth.activation(2048, K, st, seed=12, device="cuda"), g, 1e-5)], s_override=S)
    codes, sf = A.rmsnorm_quantize_activation(h, g, 1e-5, prof)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 31, 32, 127, 128, 129, 4095, 5000, 8191])
    hb = dev_bits(h[torch.from_numpy(rows).cuda()])
    oc, osf = oracle.quantize_activation(oracle.rmsnorm(hb, dev_bits(g), 1e-5), prof.perm.cpu().numpy(), S,
                                         float(prof.gs.item()))
    assert np.array_equal(codes.cpu().numpy()[rows], oc)
    Kp = prof_kp(K, S)
    sfn = sf.cpu().numpy()
    for i, m in enumerate(rows):
        for c in range(Kp // 16):
            assert sfn[oracle.sf_offset(int(m), c, Kp)] == osf[oracle.sf_offset(i, c, Kp)]


@pytest.mark.parametrize("M,N,K,S", [(16, 256, 256, 16), (200, 600, 4096, 128), (16, 4096, 14336, 128)])
def test_linear_rmsnorm_parity(A, M, N, K, S):
    st, h, g = _inputs(M, K, S, seed=N)
    w = synth.weight(N, K, seed=N + 1, device="cuda")
    prof = A.calibrate([A.rmsnorm(synth.activation(256, K, st, seed=5, device="cuda"), g, 1e-5)], s_override=S)
    qw = A.quantize_weight(w, prof)
    y = A.linear_rmsnorm(h, g, 1e-5, prof, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    perm, gs, gs_w = prof.perm.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item())
    ac, asf = oracle.quantize_activation(oracle.rmsnorm(dev_bits(h), dev_bits(g), 1e-5), perm, S, gs)
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, S, gs_w)
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
    err = np.abs(y.cpu().numpy().astype(np.float64) - yref)
    assert (err <= bound).all(), f"worst err/bound {np.max(err / np.maximum(bound, 1e-300))}"


@pytest.mark.parametrize("M,K", [(7, 48), (64, 4096), (20, 14336)])
@pytest.mark.parametrize("eps", [1e-5, 0.0])
def test_rmsnorm_vs_float64_formula(A, M, K, eps):
    """arc_rmsnorm against the float64 LLaMA RMSNorm of the same bf16 inputs, independent of any
    reduction order: within the two bf16 roundings (2^-8 each) plus fp32 rounding of the scale."""
    st, h, g = _inputs(M, K, 16, seed=5 * K + M)
    y = A.rmsnorm(h, g, eps).float().cpu().numpy().astype(np.float64)
    hf, gf = h.float().cpu().numpy().astype(np.float64), g.float().cpu().numpy().astype(np.float64)
    ref = gf * hf / np.sqrt((hf ** 2).mean(axis=1, keepdims=True) + np.float64(np.float32(eps)))
    assert np.all(np.abs(y - ref) <= np.abs(ref) * (2.0 ** -7 + 2.0 ** -15) + 1e-30)


@pytest.mark.parametrize("K", [48, 4096, 14336])
def test_rmsnorm_exact_rows_ieee(A, K):
    """On rows whose sum of squares is exact in fp32 (any order), arc_rmsnorm's bits equal the
    order-independent IEEE div / sqrt / div + two bf16 roundings computed with numpy/torch."""
    from test_oracle_rmsnorm import _exact_rows, _ieee_rmsnorm_of_exact_rows
    x = _exact_rows(33, K, seed=K + 1)
    g = synth.rmsnorm_weight(K, seed=K, device="cpu")
    y = A.rmsnorm(x.cuda(), g.cuda(), 1e-5)
    torch.cuda.synchronize()
    assert np.array_equal(dev_bits(y), _ieee_rmsnorm_of_exact_rows(x, g, 1e-5))
