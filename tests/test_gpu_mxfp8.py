"""GPU parity of the Fig.8a comparison path (plain MXFP8; Eq.3):
arc_quantize_mxfp8 is bit-exact against the oracle's MXFP8 comparator (codes and every valid scale byte)
and arc_gemm_mxfp8 (tcgen05 kind::mxf8f6f4, UE8M0 scales, K = 32 per MMA, scale byte ids per MMA) is within
the north_star bound 1e-5 * sum|a_i b_i| of the oracle's exact MXFP8 GEMM -- prefill tiles, ragged M / N /
K (K padded to 128) and the decode split-K path."""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_07475_b200 import synth
from _helpers import dev_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2601_07475_b200 import arc
    assert arc.device_supported()
    return arc


def _mask(rows, K8):
    m = np.zeros((oracle.sf_rows_padded(rows) * K8 // 32,), bool)
    for r in range(rows):
        for b in range(K8 // 32):
            m[oracle.sf_offset(r, b, K8 // 2)] = True
    return m


@pytest.mark.parametrize("M,K", [(1, 32), (7, 160), (130, 4096), (300, 14336), (64, 4128)])
def test_quantize_mxfp8_bit_exact(A, M, K):
    st = synth.Structure(K, 16 if K >= 16 else 0, seed=K)
    x = synth.activation(M, K, st, seed=M + K, device="cuda")
    codes, sf = A.quantize_mxfp8(x)
    torch.cuda.synchronize()
    oc, osf = oracle.quantize_mxfp8(dev_bits(x))
    assert np.array_equal(codes.cpu().numpy(), oc)
    mk = _mask(M, oracle.kp8(K))
    assert np.array_equal(sf.cpu().numpy()[mk], osf[mk])


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (256, 512, 4096), (200, 300, 1056), (16, 4096, 4096),
                                   (1, 256, 256), (1000, 768, 2048), (64, 1024, 14336)])
def test_gemm_mxfp8_vs_oracle(A, M, N, K):
    st = synth.Structure(K, 16, seed=N)
    x = synth.activation(M, K, st, seed=M + 1, device="cuda")
    w = synth.weight(N, K, seed=N + 1, device="cuda")
    ac, asf = A.quantize_mxfp8(x)
    bc, bsf = A.quantize_mxfp8(w)
    y = A.gemm_mxfp8(ac, asf, bc, bsf, K, out_dtype=torch.float32)
    y16 = A.gemm_mxfp8(ac, asf, bc, bsf, K)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, M - 1], np.arange(0, M, max(1, M // 24))])).astype(np.int64)
    with oracle.openmp():
        yref, bound = oracle.gemm_mxfp8_reference(ac.cpu().numpy(), asf.cpu().numpy(), bc.cpu().numpy(),
                                                  bsf.cpu().numpy(), rows=rows)
    got = y.cpu().numpy().astype(np.float64)[rows]
    err = np.abs(got - yref)
    assert (err <= bound).all(), f"{(err > bound).sum()} out of tolerance; worst {np.max(err / np.maximum(bound, 1e-300))}"
    assert torch.equal(y16, y.to(torch.bfloat16))
