"""Pins of the oracle's MXFP4-ARC variant (the paper's MXFP4 generalisation, P:387,
Table 6; SPEC: MXFP4 => g = 32, E8M0 scale, no tensor scale; reading Q25), against
definitions evaluated independently in numpy float64:

* SPEC example: a block of 32 sevens gets scale 2 (E8M0 round-up of 7/6) and code 4.0 (3.5 ties to
  the even code);
* every block: scale = the smallest power of two >= fp32(amax/6) (alpha in [1, 2), Eq.3's E8M0
  alignment factor), every code the nearest E2M1 value of x/scale (brute force, ties to even);
* residual blocks: the second stage of the exact residual x - d v(q), so primary + residual
  reconstructs x within one residual quantum, and beats the primary alone;
* weights: outlier blocks duplicated bitwise; S = 0 reduces to plain MXFP4;
* the physical NVFP4-format bytes decode to the MX values exactly (E4M3 code of 2^(e-c), gs = 2^-c),
  so the exact GEMM over them equals the float64 MX dot products."""
import numpy as np
import pytest
import torch

import oracle

E2M1 = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])


def _decode(codes, sf, rows, K, S, c, layout=0):
    """Per row: logical element values (K+S) and their block scales (float64), via the oracle's
    documented physical map (codes nibble order, 128x4 scale layout)."""
    Kp = oracle.kp(K, S)
    nlog = (K + S) // 16
    vals = np.zeros((rows, K + S))
    scales = np.zeros((rows, K + S))
    for m in range(rows):
        for lb in range(nlog):
            pb = oracle.physical_block(lb, K, S, layout)
            code = int(sf[oracle.sf_offset(m, pb, Kp)])
            d = oracle.e4m3_value(code) * 2.0 ** c
            for i in range(16):
                byte = codes[m, (16 * pb + i) // 2]
                q = (byte >> (4 * ((16 * pb + i) % 2))) & 15
                v = E2M1[q & 7] * (-1 if q & 8 else 1)
                vals[m, 16 * lb + i] = v * d
                scales[m, 16 * lb + i] = d
    return vals, scales


def _nearest_e2m1(t):
    a = np.abs(t)
    d = np.abs(E2M1[None, :] - np.minimum(a, 6.0)[:, None])
    best = np.argmin(d, axis=1)
    # ties to the even code (argmin takes the first = lower magnitude index; fix ties)
    dd = np.sort(d, axis=1)
    tie = dd[:, 0] == dd[:, 1]
    for i in np.nonzero(tie)[0]:
        cands = np.nonzero(d[i] == dd[i, 0])[0]
        best[i] = [k for k in cands if k % 2 == 0][0]
    return np.sign(t) * E2M1[best]


def _inputs(M, K, seed, spread=True):
    from paper_2601_07475_b200 import synth
    st = synth.Structure(K, 32, seed=seed)
    x = synth.activation(M, K, st, seed=seed + 1)
    perm = np.random.default_rng(seed).permutation(K).astype(np.int32)
    return x, perm


def test_spec_example_sevens():
    x = torch.full((1, 32), 7.0).to(torch.bfloat16)
    codes, sf = oracle.quantize_mx(x, np.arange(32, dtype=np.int32), 0, 0)
    assert oracle.e4m3_value(int(sf[oracle.sf_offset(0, 0, 64)])) == 2.0
    assert np.all(codes[0, :16] == 0x66)  # 4.0 in both nibbles


@pytest.mark.parametrize("K,S", [(64, 0), (256, 32), (512, 128)])
def test_blocks_against_definition(K, S):
    x, perm = _inputs(6, K, seed=K + S)
    xf = x.float().numpy().astype(np.float64)
    c = oracle.mx_offset(float(np.abs(xf).max()))
    codes, sf = oracle.quantize_mx(x, perm, S, c)
    vals, scales = _decode(codes, sf, 6, K, S, c)
    z = xf[:, perm]  # reordered
    for m in range(6):
        for b in range(K // 32):
            blk = z[m, 32 * b:32 * b + 32]
            a = np.abs(blk).max()
            raw = float(np.float32(a) / np.float32(6.0))
            d = 2.0 ** np.ceil(np.log2(raw))
            assert np.all(scales[m, 32 * b:32 * b + 32] == d)
            assert 1.0 <= d / (a / 6.0) < 2.0
            assert np.array_equal(vals[m, 32 * b:32 * b + 32], d * _nearest_e2m1(blk / d))
            if b < S // 32:
                r = blk - vals[m, 32 * b:32 * b + 32]
                res = vals[m, K + 32 * b:K + 32 * b + 32]
                d2 = scales[m, K + 32 * b]
                if np.abs(r).max() > 0:
                    raw2 = float(np.float32(np.abs(r / d).max()) / np.float32(6.0))
                    assert d2 == d * 2.0 ** np.ceil(np.log2(raw2))
                    assert np.array_equal(res, d2 * _nearest_e2m1(r / d2))
                    assert np.all(np.abs(r - res) <= d2 + 1e-300)
                    assert np.abs(r - res).sum() <= np.abs(r).sum()


def test_weight_duplicates_and_s0():
    w, perm = _inputs(5, 256, seed=7)
    c = oracle.mx_offset(float(w.float().abs().max()))
    codes, sf = oracle.quantize_mx(w, perm, 64, c, weight=True)
    vals, scales = _decode(codes, sf, 5, 256, 64, c)
    assert np.array_equal(vals[:, 256:], vals[:, :64]) and np.array_equal(scales[:, 256:], scales[:, :64])
    c0, s0 = oracle.quantize_mx(w, perm, 0, c)
    v0, _ = _decode(c0, s0, 5, 256, 0, c)
    assert np.array_equal(v0, vals[:, :256])


def test_gemm_over_physical_bytes_equals_mx_dot_products():
    x, perm = _inputs(8, 256, seed=11)
    w, _ = _inputs(16, 256, seed=12)
    S = 64
    cx = oracle.mx_offset(float(x.float().abs().max()))
    cw = oracle.mx_offset(float(w.float().abs().max()))
    ac, asf = oracle.quantize_mx(x, perm, S, cx)
    bc, bsf = oracle.quantize_mx(w, perm, S, cw, weight=True)
    y, _ = oracle.gemm_reference(ac, asf, bc, bsf, 2.0 ** -cx, 2.0 ** -cw)
    va, _ = _decode(ac, asf, 8, 256, S, cx)
    vb, _ = _decode(bc, bsf, 16, 256, S, cw)
    assert np.allclose(y, va @ vb.T, rtol=0, atol=1e-9 * np.abs(va).max() * np.abs(vb).max() * 320)


def test_out_of_range_blocks_flush():
    """Reading Q25b: a block 2^-30 below the tensor's range gets the smallest scale 2^(c-9) (E4M3
    code 0x01) and codes that match it: x / 2^(c-9) rounds to 0 here, so it dequantizes to 0."""
    x = torch.zeros(1, 64)
    x[0, 0] = 1e6
    x[0, 40] = 1e-6
    c = oracle.mx_offset(1e6)
    assert c == int(np.ceil(np.log2(np.float32(1e6) / 6))) - 8
    codes, sf = oracle.quantize_mx(x.to(torch.bfloat16), np.arange(64, dtype=np.int32), 0, c)
    vals, scales = _decode(codes, sf, 1, 64, 0, c)
    assert np.all(scales[0, 32:] == 2.0 ** (c - 9)) and np.all(vals[0, 32:] == 0.0)
    assert vals[0, 0] == _nearest_e2m1(np.array([1e6 / 2.0 ** (c + 8)]))[0] * 2.0 ** (c + 8)


def test_out_of_range_blocks_saturate():
    """Reading Q25b: a block above the offset's range (runtime max above the calibrated one) gets the
    largest scale 2^(c+8) and saturated codes +-6: every element dequantizes to sign * 6 * 2^(c+8)
    (clip), never to a shrunken value."""
    x = torch.zeros(2, 32)
    x[0, :] = 3e6
    x[1, ::2] = -5e5
    xb = x.to(torch.bfloat16)
    c = oracle.mx_offset(1e3)
    codes, sf = oracle.quantize_mx(xb, np.arange(32, dtype=np.int32), 0, c)
    vals, scales = _decode(codes, sf, 2, 32, 0, c)
    assert np.all(scales == 2.0 ** (c + 8))
    assert np.all(vals[0] == 6.0 * 2.0 ** (c + 8))
    assert np.all(vals[1, ::2] == -6.0 * 2.0 ** (c + 8)) and np.all(vals[1, 1::2] == 0.0)


def test_out_of_range_residual_clamped():
    """Outlier (residual) blocks: the residual's absolute exponent e + e2 is clamped too, so the
    dequantized primary + residual never exceeds what the clamped scales can represent, and an
    in-range block next to an out-of-range one is unaffected."""
    x = torch.zeros(1, 64)
    x[0, :32] = torch.linspace(-3e6, 2e6, 32)
    x[0, 32:] = torch.linspace(-700, 900, 32)
    xb = x.to(torch.bfloat16)
    c = oracle.mx_offset(1e3)
    codes, sf = oracle.quantize_mx(xb, np.arange(64, dtype=np.int32), 64, c)
    vals, scales = _decode(codes, sf, 1, 64, 64, c)
    assert np.all(scales[0] <= 2.0 ** (c + 8)) and np.all(scales[0] >= 2.0 ** (c - 9))
    xf = xb.float().numpy().astype(np.float64)[0]
    # in-range block 1: primary + residual within half a residual quantum of x (Q25's definition)
    rec = vals[0, 32:64] + vals[0, 96:128]
    assert np.all(np.abs(rec - xf[32:]) <= scales[0, 96:128] * 0.5 + 1e-9 * np.abs(xf[32:]))
