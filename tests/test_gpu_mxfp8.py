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


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (256, 512, 4096), (200, 300, 1056), (16, 4096, 4096),
                                   (1000, 768, 2048)])
def test_gemm_w4a8_vs_oracle(A, M, N, K):
    """The Fig.8a W4A8 comparator: MXFP8 activations x plain MXFP4 weights on kind::mxf8f6f4 with the
    weight unpacked to one byte per element by the TMA, within the north_star bound of the oracle's exact
    W4A8 GEMM; the weights come from arc_quantize_mx_native (S = 0, identity order), bit-exact vs the oracle."""
    st = synth.Structure(K, 16, seed=N + 7)
    x = synth.activation(M, K, st, seed=M + 3, device="cuda")
    w = synth.weight(N, K, seed=N + 5, device="cuda")
    ac, asf = A.quantize_mxfp8(x)
    prof = A.profile_from(np.arange(K, dtype=np.int32), 0, 1.0)
    bc, bsf = A.quantize_mx_native(w, prof, weight=True)
    obc, obsf = oracle.quantize_mx_native(dev_bits(w), np.arange(K, dtype=np.int32), 0, weight=True)
    assert np.array_equal(bc.cpu().numpy(), obc)
    y = A.gemm_w4a8(ac, asf, bc, bsf, K, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, M - 1], np.arange(0, M, max(1, M // 24))])).astype(np.int64)
    with oracle.openmp():
        yref, bound = oracle.gemm_w4a8_reference(ac.cpu().numpy(), asf.cpu().numpy(), obc, obsf, rows=rows)
    err = np.abs(y.cpu().numpy().astype(np.float64)[rows] - yref)
    assert (err <= bound).all(), f"{(err > bound).sum()} out of tolerance; worst {np.max(err / np.maximum(bound, 1e-300))}"


@pytest.mark.gpu
def test_u4_unpack_tma_layout(A):
    """The W4A8 B operand's TMA form (16U4_ALIGN16B): the load completes `rows * 64` (packed) transaction
    bytes, not the 128 bytes per row it places in shared memory, and each 16-element group lands as its 8
    packed code bytes at a 16-byte-aligned offset (the kernel's expect_tx and stage geometry rely on both)."""
    rows = 8
    g = torch.Generator().manual_seed(5)
    packed = torch.randint(0, 256, (rows, 64), generator=g, dtype=torch.uint8)
    st, buf = A.probe_u4_unpack(packed.cuda())
    assert st.tolist() == [1, 0]
    sm = buf[0, : rows * 128].view(rows, 8, 16)
    assert torch.equal(sm[:, :, :8].reshape(rows, 64), packed)
