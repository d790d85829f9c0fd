"""Oracle pins for fp16 inputs (SURVEY 8(b) arc_dtype_t ARC_FP16): the oracle's IEEE binary16 decode equals
numpy's float16 on all 2^16 bit patterns, and quantizing an fp16 tensor equals quantizing the same values
given as bf16 whenever those values are exactly representable in bf16 (the STAGE arithmetic sees identical
fp32 inputs); calibration abs-max equals numpy's |max| of the decoded values."""
import numpy as np

import oracle


def test_f16_decode_all_patterns():
    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    want = bits.view(np.float16).astype(np.float32)
    got = np.array([oracle.f16_to_f32(int(b)) for b in bits], dtype=np.float32)
    fin = np.isfinite(want)
    assert np.array_equal(got[fin], want[fin])
    assert np.array_equal(np.isnan(got), np.isnan(want)) and np.array_equal(np.isinf(got), np.isinf(want))


def test_fp16_quantize_equals_bf16_on_shared_values():
    rng = np.random.default_rng(0)
    M, K, S = 8, 256, 32
    # values exactly representable in both formats: small integers times powers of two (8 significant bits)
    v = (rng.integers(-255, 256, size=(M, K)) * np.exp2(rng.integers(-12, 3, size=(M, K)))).astype(np.float32)
    v[:, rng.choice(K, 16, replace=False)] *= 64.0  # outlier channels
    f16 = v.astype(np.float16)
    assert np.array_equal(f16.astype(np.float32), v)
    bf = (v.view(np.uint32) >> 16).astype(np.uint16)
    assert np.array_equal((bf.astype(np.uint32) << 16).view(np.float32), v)
    perm = rng.permutation(K).astype(np.int32)
    gs = float(np.float32(2688.0) / np.float32(np.abs(v).max()))
    for layout in (0, 1):
        c1, s1 = oracle.quantize_activation(f16.view(np.uint16), perm, S, gs, layout, fp16=True)
        c2, s2 = oracle.quantize_activation(bf, perm, S, gs, layout)
        assert np.array_equal(c1, c2) and np.array_equal(s1, s2)
        w1 = oracle.quantize_weight(f16.view(np.uint16), perm, S, gs, layout, fp16=True)
        w2 = oracle.quantize_weight(bf, perm, S, gs, layout)
        assert all(np.array_equal(a, b) for a, b in zip(w1, w2))


def test_fp16_calib_absmax():
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((64, 128)) * 30).astype(np.float16)
    cm = oracle.calib_absmax(x.view(np.uint16), fp16=True)
    assert np.array_equal(cm, np.abs(x.astype(np.float32)).max(axis=0))
    # the switch is scoped: a following bf16 call decodes bf16 again
    b = np.full((2, 16), 0x3F80, np.uint16)  # bf16 1.0
    assert np.array_equal(oracle.calib_absmax(b), np.ones(16, np.float32))
