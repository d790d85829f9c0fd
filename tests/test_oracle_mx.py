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


# ----------------------------------------------------------------------------- native MX format (f3)
def _decode_native(codes, sf, rows, K, S, layout=0):
    """Logical values (K+S per row) of the native MX physical format, from the documented map: 32-block
    l -> physical 2l / l+ns / 2(l-nb)+1 (interleaved) or l (contiguous), UE8M0 byte b -> 2^(b-127)."""
    Km = oracle.kpm(K, S)
    nb, ns = K // 32, S // 32
    vals = np.zeros((rows, K + S))
    for m in range(rows):
        for lb in range((K + S) // 32):
            if layout == 1:
                pb = lb
            else:
                pb = 2 * lb if lb < ns else (lb + ns if lb < nb else 2 * (lb - nb) + 1)
            d = 2.0 ** (int(sf[oracle.sf_offset(m, pb, Km // 2)]) - 127)
            for i in range(32):
                byte = codes[m, (32 * pb + i) // 2]
                q = (byte >> (4 * ((32 * pb + i) % 2))) & 15
                vals[m, 32 * lb + i] = E2M1[q & 7] * (-1 if q & 8 else 1) * d
    return vals


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("weight", [False, True])
def test_native_equals_nvfp4_format_in_range(layout, weight):
    """Within the offset's 18 binades the native MX format (UE8M0 per 32-block) and the NVFP4-format MX
    representation (E4M3 codes of 2^(e-c)) decode to the same values, element by element."""
    x, perm = _inputs(6, 256, seed=21 + layout)
    S = 64
    c = oracle.mx_offset(float(x.float().abs().max()))
    a, asf = oracle.quantize_mx(x, perm, S, c, weight=weight, layout=layout)
    v_nv, _ = _decode(a, asf, 6, 256, S, c, layout)
    n, nsf = oracle.quantize_mx_native(x, perm, S, weight=weight, layout=layout)
    v_na = _decode_native(n, nsf, 6, 256, S, layout)
    assert np.array_equal(v_na, v_nv)


def test_native_wide_range_is_the_unclamped_definition():
    """Beyond E4M3's range for any one offset (blocks 2^60 apart) the native format still holds the
    definition exactly: scale = smallest power of two >= RN(amax/6), codes = nearest E2M1 of x / scale,
    residual = the same stage on x/scale - v(q)."""
    x = torch.zeros(2, 128)
    g = torch.Generator().manual_seed(3)
    x[:, :32] = torch.randn(2, 32, generator=g) * 2.0 ** 30
    x[:, 32:64] = torch.randn(2, 32, generator=g) * 2.0 ** -30
    x[:, 64:] = torch.randn(2, 64, generator=g)
    xb = x.to(torch.bfloat16)
    perm = np.arange(128, dtype=np.int32)
    codes, sf = oracle.quantize_mx_native(xb, perm, 32)
    vals = _decode_native(codes, sf, 2, 128, 32)
    xf = xb.float().numpy().astype(np.float64)
    for m in range(2):
        for b in range(4):
            z = xf[m, 32 * b:32 * b + 32]
            s = 2.0 ** np.ceil(np.log2(np.float32(np.abs(z).max() / np.float32(6.0))))
            want = _nearest_e2m1(z / s) * s
            assert np.array_equal(vals[m, 32 * b:32 * b + 32], want), (m, b)
        # residual of outlier block 0
        z = xf[m, :32]
        s = 2.0 ** np.ceil(np.log2(np.float32(np.abs(z).max() / np.float32(6.0))))
        r = z / s - _nearest_e2m1(z / s)
        s2 = 2.0 ** np.ceil(np.log2(np.float32(np.abs(r).max() / np.float32(6.0))))
        assert np.array_equal(vals[m, 128:160], _nearest_e2m1(r / s2) * s2 * s)


def test_native_gemm_equals_float64_of_decoded():
    x, perm = _inputs(5, 256, seed=31)
    w, _ = _inputs(7, 256, seed=32)
    a, asf = oracle.quantize_mx_native(x, perm, 64)
    b, bsf = oracle.quantize_mx_native(w, perm, 64, weight=True)
    y, bound = oracle.gemm_mx_native_reference(a, asf, b, bsf)
    va = _decode_native(a, asf, 5, 256, 64)
    vb = _decode_native(b, bsf, 7, 256, 64)
    assert np.allclose(y, va @ vb.T, rtol=1e-12, atol=1e-300)
