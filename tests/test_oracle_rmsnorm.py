"""Pins of the oracle's RMSNorm (the RMSNorm stage of the paper's Fused Quantization Kernel,
PAPER.md P:164, Fig.8b; reduction order and roundings = DESIGN.md reading Q23) against
what the mathematics fixes, independent of the oracle's own formula:

* float64 RMSNorm of the same bf16 inputs, within the two bf16 roundings;
* exact invariance of every output bit under scaling a row by a power of two (eps = 0):
  each step of the pinned order commutes with the scaling, so any wrong normalisation
  (missing square root, mean of |x|, wrong divisor) or a dropped scale breaks it;
* constant rows normalise to +-1 exactly (g = 1, eps = 0), for power-of-two and ragged K;
* torch's fp32 RMSNorm (its own reduction order, rsqrt) within one bf16 ulp;
* non-finite input is an error."""
import numpy as np
import pytest
import torch

import oracle


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def _f(bits: np.ndarray) -> np.ndarray:
    return torch.from_numpy(bits.astype(np.int16)).view(torch.bfloat16).float().numpy().astype(np.float64)


def _rows(M, K, seed, outliers=True):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(M, K, generator=g) * torch.exp(0.5 * torch.randn(M, 1, generator=g))
    if outliers:
        idx = torch.randperm(K, generator=g)[: max(1, K // 64)]
        x[:, idx] *= 50.0
    gamma = 1.0 + 0.2 * torch.randn(K, generator=g)
    return x.to(torch.bfloat16), gamma.to(torch.bfloat16)


@pytest.mark.parametrize("K", [16, 48, 256, 4096, 14336])
@pytest.mark.parametrize("eps", [0.0, 1e-5, 1.0])
def test_matches_float64_formula(K, eps):
    x, g = _rows(8, K, seed=K)
    y = _f(oracle.rmsnorm(x, g, eps))
    xf, gf = _f(_bits(x)), _f(_bits(g))
    ref = gf * xf / np.sqrt((xf ** 2).mean(axis=1, keepdims=True) + np.float64(np.float32(eps)))
    # two bf16 roundings (unit roundoff 2^-8 each: 7 stored mantissa bits) + fp32 scale rounding
    assert np.all(np.abs(y - ref) <= np.abs(ref) * (2.0 ** -7 + 2.0 ** -15) + 1e-30)


@pytest.mark.parametrize("K", [64, 80, 4096])
@pytest.mark.parametrize("k", [-4, 3, 7])
def test_power_of_two_scale_invariance(K, k):
    x, g = _rows(6, K, seed=100 + K)
    xs = (x.float() * 2.0 ** k).to(torch.bfloat16)  # exact: power-of-two scaling of bf16
    assert torch.equal(xs.float(), x.float() * 2.0 ** k)
    assert np.array_equal(oracle.rmsnorm(x, g, 0.0), oracle.rmsnorm(xs, g, 0.0))


@pytest.mark.parametrize("K", [16, 48, 4096, 4112])
@pytest.mark.parametrize("c", [3.0, -0.375, 1.5e-3, 2.0 ** 20])
def test_constant_rows_normalise_to_one(K, c):
    x = torch.full((2, K), c).to(torch.bfloat16)
    g = torch.ones(K, dtype=torch.bfloat16)
    y = _f(oracle.rmsnorm(x, g, 0.0))
    assert np.all(y == np.sign(c))


def test_gamma_is_applied_per_channel():
    K = 64
    x = torch.full((1, K), 2.0).to(torch.bfloat16)
    g = torch.arange(K, dtype=torch.float32).to(torch.bfloat16)  # exact small integers
    y = _f(oracle.rmsnorm(x, g, 0.0))
    assert np.array_equal(y[0], _f(_bits(g)))


def test_torch_fp32_rmsnorm_within_one_ulp():
    """Third-party check: the HF LLaMA RMSNorm formula evaluated by torch in fp32."""
    x, g = _rows(16, 4096, seed=7)
    eps = 1e-5
    h = x.float()
    var = h.pow(2).mean(-1, keepdim=True)
    ref = (g * (h * torch.rsqrt(var + eps)).to(torch.bfloat16)).to(torch.bfloat16)
    y = oracle.rmsnorm(x, g, eps).astype(np.int32)
    r = _bits(ref).astype(np.int32)
    # same sign -> the bf16 bit patterns differ by the ulp distance
    assert np.abs(y - r).max() <= 1


def test_scale_is_the_reciprocal_rms():
    x, _ = _rows(1, 256, seed=3)
    r = oracle.rmsnorm_scale(_bits(x)[0], 1e-5)
    xf = _f(_bits(x))[0]
    assert abs(r * np.sqrt((xf ** 2).mean() + 1e-5) - 1.0) < 2e-6


def test_nonfinite_is_an_error():
    x, g = _rows(2, 64, seed=1)
    x[1, 5] = float("inf")
    with pytest.raises(oracle.OracleError):
        oracle.rmsnorm(x, g, 1e-5)
    with pytest.raises(oracle.OracleError):  # all-zero row with eps = 0 -> 1/0
        oracle.rmsnorm(torch.zeros(1, 64, dtype=torch.bfloat16), g, 0.0)


def _exact_rows(M, K, seed):
    """Rows of n * 2^-3 with |n| <= 15: every square is a multiple of 2^-6 and every partial sum of
    squares stays below 2^24 * 2^-6, so the fp32 sum of squares is exact in ANY order."""
    rng = np.random.default_rng(seed)
    n = rng.integers(-15, 16, size=(M, K)).astype(np.float32)
    n[:, 0] = 7.0  # no all-zero row
    return torch.from_numpy(n * np.float32(0.125)).to(torch.bfloat16)


def _ieee_rmsnorm_of_exact_rows(x: torch.Tensor, g: torch.Tensor, eps: float) -> np.ndarray:
    """Order-independent definition of reading Q23 on exact rows: ss exact (float64 sum == fp32 sum),
    mean = RN32(ss / K), r = RN32(1 / RN32(sqrt(RN32(mean + eps)))), y = bf16(g * bf16(x * r)) with
    RN-even bf16 roundings done by torch's float32 -> bfloat16 cast (a third-party rounding)."""
    xf = x.float().numpy()
    K = xf.shape[1]
    ss64 = (xf.astype(np.float64) ** 2).sum(axis=1)
    ss = ss64.astype(np.float32)
    assert np.array_equal(ss.astype(np.float64), ss64)           # the sum really is exact in fp32
    mean = ss / np.float32(K)
    r = np.float32(1.0) / np.sqrt(mean + np.float32(eps))
    assert r.dtype == np.float32
    t = torch.from_numpy(xf * r[:, None]).to(torch.bfloat16).float()
    y = (g.float()[None, :] * t).to(torch.bfloat16)
    return _bits(y)


@pytest.mark.parametrize("K", [16, 48, 256, 1040, 4096, 14336])
@pytest.mark.parametrize("eps", [0.0, 1e-5, 1e-6])
def test_exact_rows_match_order_independent_ieee(K, eps):
    """The oracle's reduction order (Q23: 32 round-robin partials + pairwise trees, chosen
    in 036374d to suit the kernel's conflict-free loads) is a decision; the arithmetic after the
    reduction is not.  On rows whose sum of squares is exact in fp32 the order cannot matter, so the
    oracle's bits must equal the IEEE div / sqrt / div and the two bf16 roundings computed here
    independently with numpy float32 (each op correctly rounded) and torch's bf16 cast."""
    x = _exact_rows(9, K, seed=K)
    _, g = _rows(1, K, seed=K + 1)
    assert np.array_equal(oracle.rmsnorm(x, g, eps), _ieee_rmsnorm_of_exact_rows(x, g, eps))


def test_exact_rows_scale_is_ieee_reciprocal_sqrt():
    x = _exact_rows(4, 4096, seed=5)
    for i in range(4):
        xf = x[i].float().numpy()
        ss = np.float32((xf.astype(np.float64) ** 2).sum())
        want = np.float32(1.0) / np.sqrt(ss / np.float32(4096) + np.float32(1e-5))
        assert np.float32(oracle.rmsnorm_scale(_bits(x[i:i + 1])[0], 1e-5)) == want
