"""Pins of the oracle's plain-MXFP8 comparator format (the Fig.8a comparison GEMMs, P:375 / P:395; Eq.3's
single MXFP8 stage): every 32-block's scale is the smallest power of two >= amax/448 (alpha_mx in
[1, 2), against Eq.3's own comparator or_mxfp8_block), every code the nearest E4M3 value of x / scale (brute
force over all 256 codes decoded by torch's float8_e4m3fn, ties to the even code), pad blocks zero, and the
exact MXFP8 GEMM equals the float64 dot products of the independently decoded operands."""
import numpy as np
import pytest
import torch

import oracle


def _x(M, K, seed, spread=8.0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(M, K, generator=g) * torch.exp(spread * torch.rand(M, K // 32, generator=g)).repeat_interleave(32, 1)
    return x.to(torch.bfloat16)


E4M3 = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).float().numpy().astype(np.float64)


def _decode(codes, sf, M, K8):
    vals = E4M3[codes.astype(np.int64)]
    sc = np.zeros((M, K8 // 32))
    for m in range(M):
        for b in range(K8 // 32):
            sc[m, b] = 2.0 ** (int(sf[oracle.sf_offset(m, b, K8 // 2)]) - 127)
    return vals * np.repeat(sc, 32, axis=1), sc


@pytest.mark.parametrize("M,K", [(5, 32), (3, 160), (130, 256)])
def test_scales_and_codes_brute_force(M, K):
    x = _x(M, K, seed=K + M)
    codes, sf = oracle.quantize_mxfp8(x)
    K8 = oracle.kp8(K)
    assert K8 % 128 == 0 and codes.shape == (M, K8)
    xf = x.float().numpy().astype(np.float64)
    _, sc = _decode(codes, sf, M, K8)
    finite = np.isfinite(E4M3)
    for m in range(M):
        for b in range(K8 // 32):
            if b * 32 >= K:  # pad block: zero codes, scale 1
                assert sc[m, b] == 1.0 and not codes[m, b * 32:(b + 1) * 32].any()
                continue
            z = xf[m, b * 32:(b + 1) * 32]
            s_eq3, _ = oracle.mxfp8_block(z.astype(np.float32))
            assert sc[m, b] == s_eq3
            amax = np.abs(z).max()
            assert amax == 0 or 1.0 <= sc[m, b] * 448 / np.float32(amax / 448) / 448 < 2.0 + 1e-12
            for i in range(32):
                t = z[i] / sc[m, b]
                d = np.where(finite, np.abs(E4M3 - t), np.inf)
                best = np.flatnonzero(d == d.min())
                got = int(codes[m, b * 32 + i])
                assert got in best, (m, b, i)
                if best.size > 1:  # tie: the even mantissa code (same sign class as t)
                    assert (got & 1) == 0


def test_gemm_exact_equals_float64_of_decoded():
    M, N, K = 6, 9, 320
    a, asf = oracle.quantize_mxfp8(_x(M, K, seed=1))
    b, bsf = oracle.quantize_mxfp8(_x(N, K, seed=2))
    K8 = oracle.kp8(K)
    y, bound = oracle.gemm_mxfp8_reference(a, asf, b, bsf)
    va, _ = _decode(a, asf, M, K8)
    vb, _ = _decode(b, bsf, N, K8)
    ref = va @ vb.T
    assert np.allclose(y, ref, rtol=1e-12, atol=0)
    assert np.all(bound >= 0) and np.all(np.abs(y) <= bound * 1e5 * (1 + 1e-12))
    with oracle.openmp():
        y2, _ = oracle.gemm_mxfp8_reference(a, asf, b, bsf)
        a2, asf2 = oracle.quantize_mxfp8(_x(M, K, seed=1))
    assert np.array_equal(y, y2) and np.array_equal(a, a2) and np.array_equal(asf, asf2)


def test_w4a8_gemm_exact_equals_float64_of_decoded():
    """Fig.8a W4A8 comparator: MXFP8 activations x plain MXFP4 weights (native MX format, S = 0,
    identity order); the exact GEMM equals float64 dot products of the independently decoded operands."""
    M, N, K = 5, 7, 288
    a, asf = oracle.quantize_mxfp8(_x(M, K, seed=3))
    w = _x(N, K, seed=4)
    b, bsf = oracle.quantize_mx_native(w, np.arange(K, dtype=np.int32), 0, weight=True)
    K8 = oracle.kp8(K)
    assert oracle.kpm(K, 0) == K8
    y, bound = oracle.gemm_w4a8_reference(a, asf, b, bsf)
    va, _ = _decode(a, asf, M, K8)
    E2M1 = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    vb = np.zeros((N, K8))
    for n in range(N):
        for p in range(K8):
            q = (b[n, p // 2] >> (4 * (p % 2))) & 15
            vb[n, p] = E2M1[q & 7] * (-1 if q & 8 else 1) * 2.0 ** (int(bsf[oracle.sf_offset(n, p // 32, K8 // 2)]) - 127)
    assert np.allclose(y, va @ vb.T, rtol=1e-12, atol=1e-300)
