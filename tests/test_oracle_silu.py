"""Pins of the oracle's SiLU-mul stage (the producer of the down-projection input site of the
paper's decoder layer, Fig.5; evaluation order = DESIGN.md reading Q24) against what the
mathematics fixes, independent of the oracle's own op sequence:

* every finite bf16 gate value g (all 2^16 bit patterns): the fp32 SiLU within 4 fp32 ulp of
  the long-double g / (1 + e^-g) (x87 80-bit, 64-bit significand), so a wrong sign, branch,
  constant or polynomial term fails somewhere in the sweep;
* its bf16 rounding equals the correctly rounded bf16 SiLU on every one of them;
* torch's CPU bf16 SiLU (a different exp implementation) gives the same bits wherever its
  exp(-g) does not overflow, and SiLU * up agrees;
* fixed points of the function: SiLU(0) = 0, SiLU(g) = g in bf16 for large g, SiLU -> -0 for
  very negative g; non-finite input and inconsistent shapes are errors."""
import numpy as np
import pytest
import torch

import oracle

LD = np.longdouble


def _all_finite_bf16() -> np.ndarray:
    b = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    exp = (b >> 7) & 0xFF
    return b[exp != 0xFF]


def _bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _silu_ld(g32: np.ndarray) -> np.ndarray:
    g = g32.astype(LD)
    return g / (LD(1) + np.exp(-g))


def _rn_bf16_ld(v: np.ndarray) -> np.ndarray:
    """Correct round-to-nearest-even of long-double values to bf16 bits (finite, |v| < 2^128)."""
    mag = np.abs(v)
    t = (mag.astype(np.float32).view(np.uint32) >> 16).astype(np.int64)  # a neighbour (any rounding)
    cands = np.stack([np.maximum(t - 1, 0), t, t + 1])
    vals = (cands.astype(np.uint32) << 16).view(np.float32).astype(LD)
    err = np.abs(vals - mag[None, :])
    best = np.argmin(err, axis=0)
    # ties: the even pattern
    e_sorted = np.sort(err, axis=0)
    tie = e_sorted[0] == e_sorted[1]
    out = cands[best, np.arange(v.size)]
    if tie.any():
        idx = np.nonzero(tie)[0]
        for i in idx:
            m = [c for c in cands[:, i] if abs(LD(np.uint32(c << 16).view(np.float32)) - mag[i]) == e_sorted[0, i]]
            out[i] = [c for c in m if c % 2 == 0][0]
    sign = np.signbit(v).astype(np.int64) << 15
    return (out | sign).astype(np.uint16)


def _f32_to_bf16_rne(f: np.ndarray) -> np.ndarray:
    u = f.astype(np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def test_long_double_is_extended():
    assert np.finfo(LD).nmant >= 63, "the pins need x87 extended precision"


def test_silu_f32_within_4_ulp_of_long_double_everywhere():
    g = _all_finite_bf16()
    s = oracle.silu_f32(g).astype(LD)
    ref = _silu_ld(_bf16_to_f32(g))
    err = np.abs(s - ref)
    gf = np.abs(_bf16_to_f32(g))
    # E = e^-|g| is an fp32 normal for |g| < 87: a few roundings, measured max 3.02 ulp
    normal = gf < 87.0
    assert np.all(err[normal] <= LD(4) * LD(2.0) ** -24 * np.abs(ref[normal]))
    # beyond, E is denormal (absolute error <= 2^-150) or 0, and SiLU(g) = g or |SiLU(g)| < 2^-118
    assert np.all(err[~normal] <= LD(2.0) ** -142 + LD(4) * LD(2.0) ** -24 * np.abs(ref[~normal]))
    assert normal.sum() > 30000


def test_bf16_silu_is_correctly_rounded_everywhere():
    g = _all_finite_bf16()
    sb = _f32_to_bf16_rne(oracle.silu_f32(g))
    want = _rn_bf16_ld(_silu_ld(_bf16_to_f32(g)))
    # a miss would need the fp32 value within ~4 ulp of a bf16 midpoint; none of the 2^16 is
    assert np.array_equal(sb, want)


def test_torch_bf16_silu_agrees():
    g = _all_finite_bf16()
    gt = torch.from_numpy(g.astype(np.int16)).view(torch.bfloat16)
    tb = torch.nn.functional.silu(gt).view(torch.int16).numpy().view(np.uint16)
    sb = _f32_to_bf16_rne(oracle.silu_f32(g))
    gf = _bf16_to_f32(g)
    ovf = gf < -88.0  # torch evaluates x / (1 + exp(-x)): exp overflows and the result is -0
    assert np.array_equal(tb[~ovf], sb[~ovf])
    want = _rn_bf16_ld(_silu_ld(gf[ovf]))
    assert np.array_equal(sb[ovf], want)  # the E / (1 + E) form stays correctly rounded there


def test_fixed_points():
    def sb(x):
        return _f32_to_bf16_rne(oracle.silu_f32(_f32_to_bf16_rne(np.array([x], np.float32))))[0]

    assert sb(0.0) == 0x0000
    assert sb(-0.0) == 0x8000
    for x in (32.0, 100.0, 1e4, 3e38):
        assert sb(x) == _f32_to_bf16_rne(np.array([x], np.float32))[0]
    for x in (-120.0, -1e4, -3e38):
        assert sb(x) == 0x8000
    # SiLU(1) = 1/(1+e^-1) = 0.7310585786... -> bf16 0.73046875 (0x3F3B)
    assert sb(1.0) == 0x3F3B


@pytest.mark.parametrize("M,K", [(3, 16), (16, 256), (7, 4096)])
def test_silu_mul_matches_torch(M, K):
    gen = torch.Generator().manual_seed(M * 1000 + K)
    gu = (torch.randn(M, 2 * K, generator=gen) * 3.0).to(torch.bfloat16)
    h = oracle.silu_mul(gu)
    gate, up = gu[:, :K], gu[:, K:]
    ref = (torch.nn.functional.silu(gate) * up).contiguous().view(torch.int16).numpy().view(np.uint16)
    bad = np.nonzero(h != ref)
    assert bad[0].size <= max(2, M * K // 2000)
    # where the two SiLUs round differently the products differ by at most a couple of ulp
    d = np.abs(h[bad].astype(np.int64) - ref[bad].astype(np.int64))
    assert np.all(d <= 2)


def test_silu_mul_layout_arguments():
    gen = torch.Generator().manual_seed(5)
    M, K = 4, 64
    gu = torch.randn(M, 3 * K, generator=gen).to(torch.bfloat16)  # gate [0,K), pad, up [2K,3K)
    h = oracle.silu_mul(gu, K=K, up_off=2 * K)
    h2 = oracle.silu_mul(torch.cat([gu[:, :K], gu[:, 2 * K:]], dim=1))
    assert np.array_equal(h, h2)
    with pytest.raises(oracle.OracleError):
        oracle.silu_mul(gu, K=K, up_off=K - 16)


def test_non_finite_is_an_error():
    gu = torch.zeros(2, 32, dtype=torch.bfloat16)
    gu[1, 20] = float("inf")
    with pytest.raises(oracle.OracleError):
        oracle.silu_mul(gu)
