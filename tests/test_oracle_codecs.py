"""Pins for the oracle's minifloat codecs (oracle/arc_oracle.c C1/C2).

Each check compares the oracle with something other than itself: the format
parameters of Table 7, an independent bit-field decoder, a
brute-force argmin/scan over all codes, torch's float8_e4m3fn, or a SPEC.md
worked example.
"""
import numpy as np
import pytest
import torch

import oracle


def _minifloat(code, ebits, mbits, bias):
    """Independent bit-field decoder (sign | exponent | mantissa, IEEE-style subnormals)."""
    s = (code >> (ebits + mbits)) & 1
    e = (code >> mbits) & ((1 << ebits) - 1)
    m = code & ((1 << mbits) - 1)
    if e == 0:
        v = m / (1 << mbits) * 2.0 ** (1 - bias)
    else:
        v = (1 + m / (1 << mbits)) * 2.0 ** (e - bias)
    return -v if s else v


def test_e2m1_table_matches_table7():
    # Table 7: FP4 E2M1, bias 1, max normal +-6.
    vals = oracle.e2m1_values()
    ref = np.array([_minifloat(c, 2, 1, 1) for c in range(16)], np.float32)
    assert np.array_equal(vals, ref)
    assert vals.max() == 6.0 and vals.min() == -6.0
    assert np.signbit(vals[8]) and vals[8] == 0.0  # 0x8 is -0


def _e2m1_bruteforce(t):
    """argmin over all 16 codes of |v(c) - t|, clamped to +-6; ties -> even code
    (mantissa bit 0); sign of the input kept for zero."""
    mags = np.array([_minifloat(c, 2, 1, 1) for c in range(8)])
    a = min(abs(float(t)), 6.0)
    d = np.abs(mags - a)
    best = [c for c in range(8) if d[c] == d.min()]
    c = best[0] if len(best) == 1 else [b for b in best if b % 2 == 0][0]
    return c | (8 if np.signbit(t) else 0)


def test_e2m1_encode_bruteforce_random_and_ties():
    rng = np.random.default_rng(1)
    xs = np.concatenate([
        rng.uniform(-7, 7, 20000).astype(np.float32),
        rng.standard_normal(5000).astype(np.float32) * 0.3,
        np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0, 7.0, 1e9, 0.0, -0.0, -0.25, -5.0, -1e-30],
                 np.float32),
    ])
    xs = np.concatenate([xs, np.nextafter(xs, np.float32(np.inf)), np.nextafter(xs, np.float32(-np.inf))])
    got = oracle.e2m1_encode(xs)
    ref = np.array([_e2m1_bruteforce(x) for x in xs], np.uint8)
    assert np.array_equal(got, ref)


def test_e2m1_spec_example_and_worst_error():
    # 5.0 (midpoint of 4 and 6) -> 4.0 under ties-to-even.
    assert oracle.e2m1_value(int(oracle.e2m1_encode([5.0])[0])) == 4.0
    # S:73 / eps4 = 2^-2: worst |x - Q(x)| on [-6, 6] is 1.0 (half the 4..6 gap).
    grid = np.linspace(-6, 6, 200001).astype(np.float32)
    dq = oracle.e2m1_values()[oracle.e2m1_encode(grid)]
    err = np.abs(dq.astype(np.float64) - grid)
    assert err.max() <= 1.0 and err.max() > 0.9999


def test_e4m3_table_matches_table7_and_torch():
    # Table 7: FP8 E4M3, bias 7, max normal +-448.
    vals = oracle.e4m3_values()
    ref = np.array([_minifloat(c, 4, 3, 7) for c in range(256)], np.float32)
    finite = [c for c in range(256) if (c & 0x7F) != 0x7F]          # 0x7F/0xFF are NaN in E4M3FN
    assert np.array_equal(vals[finite], ref[finite])
    tv = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).float().numpy()
    assert np.array_equal(vals[finite], tv[finite])
    pos = vals[:0x7F]
    assert np.all(np.diff(pos) > 0), "127 non-negative finite codes strictly increasing"
    assert pos[1] == 2.0 ** -9 and pos[8] == 2.0 ** -6 and pos[0x7E] == 448.0


def _e4m3_ceil_bruteforce(v):
    vals = [_minifloat(c, 4, 3, 7) for c in range(0x7F)]
    if not v > 0:
        return 0
    for c, x in enumerate(vals):
        if x >= v:
            return c
    return 0x7E


def test_e4m3_ceil_bruteforce_and_alpha():
    rng = np.random.default_rng(2)
    vs = np.concatenate([
        np.exp(rng.uniform(np.log(1e-4), np.log(600.0), 30000)).astype(np.float32),
        oracle.e4m3_values()[1:0x7F], np.array([0.0, 1e-30, 448.0, 449.0, 1e6], np.float32),
    ])
    vs = np.concatenate([vs, np.nextafter(vs, np.float32(np.inf)), np.nextafter(vs, np.float32(0))])
    got = oracle.e4m3_ceil(vs)
    ref = np.array([_e4m3_ceil_bruteforce(float(v)) for v in vs], np.uint8)
    assert np.array_equal(got, ref)
    # "2^-3 step size": alpha = s/raw in [1, 1.125) on the normal range.
    normal = (vs >= 2.0 ** -6) & (vs <= 448.0)
    alpha = oracle.e4m3_values()[got[normal]].astype(np.float64) / vs[normal]
    assert alpha.min() >= 1.0 and alpha.max() < 1.125


def test_e4m3_rn_matches_torch_cast():
    rng = np.random.default_rng(3)
    xs = (rng.standard_normal(50000) * np.exp(rng.uniform(-8, 5, 50000))).astype(np.float32)
    xs = xs[np.abs(xs) <= 448]
    got = oracle.e4m3_rn(xs)
    ref = torch.from_numpy(xs).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(got, ref)


def test_e8m0_up_spec_examples():
    # 1.0 -> 1.0, 7/6 -> 2.0, 0.3 -> 0.5.
    assert oracle.e8m0_up(1.0) == 1.0
    assert oracle.e8m0_up(np.float32(7 / 6)) == 2.0
    assert oracle.e8m0_up(0.3) == 0.5
    rng = np.random.default_rng(4)
    for v in np.exp(rng.uniform(-20, 20, 2000)).astype(np.float32):
        s = oracle.e8m0_up(float(v))
        assert 1.0 <= s / float(v) < 2.0  # alpha_mx in [1, 2) (Eq.3)


def test_stage_spec_example_16_sixes():
    # 16 copies of 6.0 at gs=1 -> scale 1.0 (0x38), all codes 6.0, zero error.
    sf, d, t, q = oracle.stage([6.0] * 16, 1.0)
    assert sf == 0x38 and d == 1.0 and np.all(q == 7)


def test_stage_zero_and_subnormal_blocks():
    sf, d, t, q = oracle.stage([0.0] * 8 + [-0.0] * 8, 1.0)
    assert sf == 0 and d == 0.0 and np.all(q[:8] == 0) and np.all(q[8:] == 8)
    # max 1e-4 at gs=1: raw scale 1.67e-5 < 2^-9 -> smallest subnormal 0x01, codes round to 0
    sf, d, t, q = oracle.stage([1e-4] + [0.0] * 15, 1.0)
    assert sf == 0x01 and d == 2.0 ** -9 and q[0] == 0


def test_stage_properties_bruteforce():
    """Every STAGE output is checked against definitions evaluated in float64:
    sf is the smallest E4M3 value >= a*fl(base/6) (up to that one fp32 product
    rounding); each code is the brute-force nearest E2M1 of t; no clipping when
    the scale is not saturated (|t| <= 6)."""
    rng = np.random.default_rng(5)
    e4 = oracle.e4m3_values().astype(np.float64)
    for it in range(3000):
        z = (rng.standard_normal(16) * np.exp(rng.uniform(-6, 6))).astype(np.float32)
        base = float(np.float32(np.exp(rng.uniform(-3, 6))))
        sf, d, t, q = oracle.stage(z, base)
        a = float(np.max(np.abs(z)))
        c6 = float(np.float32(base) / np.float32(6.0))
        raw = float(np.float32(np.float32(a) * np.float32(c6)))
        if raw <= 448:
            assert e4[sf] >= raw and (sf == 0 or e4[sf - 1] < raw)
            assert np.all(np.abs(t) <= 6.0 * (1 + 2.0 ** -20))
        assert all(q[i] == _e2m1_bruteforce(t[i]) for i in range(16))
