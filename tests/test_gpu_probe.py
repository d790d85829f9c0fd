"""Hardware-semantics pins: the quantization kernel's E2M1 encoder (cvt.rn.satfinite
.e2m1x2 + sign fix-up) over ALL 2^32 fp32 bit patterns, and its E4M3 ceil encoder,
against the oracle's closed forms (readings Q1, Q2)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2601_07475_b200 import arc
    return arc


def test_e2m1_exhaustive_2pow32(A):
    chunk = 1 << 27
    for c in range(1 << 32 >> 27):
        start = c * chunk
        got = A.probe_e2m1_bits(start, chunk).cpu().numpy()
        bits = np.arange(start, start + chunk, dtype=np.uint64).astype(np.uint32)
        f = bits.view(np.float32)
        ok = ~np.isnan(f)
        ref = oracle.e2m1_encode(f[ok])
        bad = np.nonzero(got[ok] != ref)[0]
        assert bad.size == 0, f"chunk {c}: {bad.size} mismatches, first input {f[ok][bad[:4]]}"


def test_e2m1_raw_hardware_semantics(A):
    """Record how the raw cvt.rn.satfinite.e2m1x2.f32 treats the sign of values that
    round to zero, and check it is RNE with saturation everywhere else."""
    chunk = 1 << 27
    sign_mismatch = 0
    for c in range(1 << 32 >> 27):
        start = c * chunk
        got = A.probe_e2m1_raw_bits(start, chunk).cpu().numpy()
        f = np.arange(start, start + chunk, dtype=np.uint64).astype(np.uint32).view(np.float32)
        ok = ~np.isnan(f)
        ref = oracle.e2m1_encode(f[ok])
        g = got[ok]
        assert np.array_equal(g & 7, ref & 7), f"magnitude mismatch in chunk {c}"
        sign_mismatch += int(np.count_nonzero(g != ref))
    print(f"raw cvt sign mismatches vs oracle (Q1 signed zero): {sign_mismatch}")


def test_e4m3_ceil_matches_oracle(A):
    rng = np.random.default_rng(0)
    v = np.concatenate([
        np.exp(rng.uniform(np.log(1e-9), np.log(1e4), 2_000_000)).astype(np.float32),
        oracle.e4m3_values()[:0x7F], np.array([0.0, 448.0, 449.0, 1e30, 2.0 ** -10, 2.0 ** -9], np.float32)])
    v = np.concatenate([v, np.nextafter(v, np.float32(np.inf)), np.nextafter(v, np.float32(0))])
    got = A.probe_e4m3_ceil(torch.from_numpy(v).cuda()).cpu().numpy()
    assert np.array_equal(got, oracle.e4m3_ceil(v))
