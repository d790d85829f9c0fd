"""CPU tests of the C-ABI library: it loads, exports every symbol include/*.h
declares, validates arguments synchronously (before touching the device), and
its host-side outlier selection equals the oracle's."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def arc():
    from paper_2601_07475_b200 import build
    build.build()
    from paper_2601_07475_b200 import arc as A
    return A


def _declared():
    names = set()
    for h in ("arc.h", "arc_probe.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"ARC_API\s+[\w\s\*]+?\b(arc_\w+)\s*\(", src))
    return names


def test_exports_every_declared_symbol(arc):
    declared = _declared()
    assert len(declared) >= 17
    lib = ctypes.CDLL(arc.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(arc.EXPORTED)


def test_buffer_sizes(arc):
    kp, cb, sb = arc.buffer_sizes(16, 256, 16)
    assert (kp, cb, sb) == (320, 16 * 160, 128 * 20)
    kp, cb, sb = arc.buffer_sizes(2048, 4096, 128)
    assert (kp, cb, sb) == (4224, 2048 * 2112, 2048 * 264)
    for K, S in ((0, 0), (24, 0), (32, 8), (32, 48), (32, -16)):
        with pytest.raises(arc.ArcError) as e:
            arc.buffer_sizes(1, K, S)
        assert e.value.status == 2


def test_validation_is_synchronous(arc):
    lib = arc.lib()
    P = ctypes.c_void_p
    fake = P(0x10000)
    prof = arc.ArcProfile(256, 16, 0x10000, 0x10000, 0)
    # null pointers -> ARC_ERR_NULL
    assert lib.arc_quantize_activation(None, 4, 256, ctypes.byref(prof), fake, fake, None) == 1
    # bad S -> ARC_ERR_SHAPE
    bad = arc.ArcProfile(256, 8, 0x10000, 0x10000, 0)
    assert lib.arc_quantize_activation(fake, 4, 256, ctypes.byref(bad), fake, fake, None) == 2
    # misaligned -> ARC_ERR_ALIGN
    assert lib.arc_quantize_activation(P(0x10008), 4, 256, ctypes.byref(prof), fake, fake, None) == 3
    # ldx < K -> ARC_ERR_SHAPE
    assert lib.arc_quantize_activation(fake, 4, 128, ctypes.byref(prof), fake, fake, None) == 2
    # qweight Kp mismatch -> ARC_ERR_SHAPE
    qw = arc.ArcQWeight(64, 256, 256, 16, 0, 0x10000, 0x10000, 0x10000)
    assert lib.arc_gemm(fake, fake, fake, 4, ctypes.byref(qw), fake, 0, 64, None, 0, None) == 2
    # workspace too small -> ARC_ERR_WORKSPACE
    qw = arc.ArcQWeight(64, 256, 320, 16, 0, 0x10000, 0x10000, 0x10000)
    assert lib.arc_linear(fake, 4, 256, ctypes.byref(prof), ctypes.byref(qw), fake, 0, 64, fake, 16, None) == 5
    # profile / qweight disagreement -> ARC_ERR_SHAPE
    qw2 = arc.ArcQWeight(64, 256, 320, 16, 1, 0x10000, 0x10000, 0x10000)
    assert lib.arc_linear(fake, 4, 256, ctypes.byref(prof), ctypes.byref(qw2), fake, 0, 64, fake, 1 << 20,
                          None) == 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal path")
def test_no_fallback_without_sm100(arc):
    """With valid arguments but no sm_100 device the library refuses (ARC_ERR_UNSUPPORTED)."""
    lib = arc.lib()
    fake = ctypes.c_void_p(0x10000)
    prof = arc.ArcProfile(256, 16, 0x10000, 0x10000, 0)
    assert lib.arc_device_supported() == 0
    assert lib.arc_quantize_activation(fake, 4, 256, ctypes.byref(prof), fake, fake, None) == 4
    qw = arc.ArcQWeight(64, 256, 320, 16, 0, 0x10000, 0x10000, 0x10000)
    assert lib.arc_gemm(fake, fake, fake, 4, ctypes.byref(qw), fake, 0, 64, fake, 1 << 20, None) == 4


def test_select_outliers_matches_oracle(arc):
    import oracle
    rng = np.random.default_rng(0)
    for _ in range(40):
        K = int(rng.integers(1, 64)) * 16
        cm = (np.exp(rng.uniform(-4, 4, K)) * (rng.random(K) < 0.8)).astype(np.float32)
        cm[rng.integers(0, K, 4)] = cm[rng.integers(0, K)]
        a = arc.select_outliers(cm)
        o = oracle.select_outliers(cm)
        assert np.array_equal(a["perm"], o["perm"])
        for k in ("S", "S_raw", "M", "tau", "gs"):
            assert a[k] == o[k], k
    with pytest.raises(arc.ArcError):
        arc.select_outliers(np.array([np.nan] + [1.0] * 15, np.float32))


def test_gather_order_keeps_block_sets(arc):
    """arc_gather_order only permutes channels inside each 16-block (reading Q22)."""
    rng = np.random.default_rng(3)
    for K in (16, 256, 4096, 14336):
        perm = rng.permutation(K).astype(np.int32)
        out = arc.gather_order(perm)
        assert sorted(out.tolist()) == list(range(K))
        for b in range(K // 16):
            assert set(out[16 * b:16 * b + 16]) == set(perm[16 * b:16 * b + 16])
        assert np.array_equal(out, arc.gather_order(perm))  # deterministic
    with pytest.raises(arc.ArcError):
        arc.gather_order(np.zeros(32, np.int32))


def test_validation_of_producer_and_mx_entry_points(arc):
    """Argument checks of the fused-producer, SwiGLU, MXFP4-ARC and gather-order entry points run
    before any device work (no GPU needed)."""
    lib = arc.lib()
    P = ctypes.c_void_p
    fake = P(0x10000)
    prof = arc.ArcProfile(256, 16, 0x10000, 0x10000, 0)
    # SiLU-mul: up_off < K -> ARC_ERR_SHAPE; pairs need ld >= 2K
    assert lib.arc_silu_mul(fake, 4, 256, 512, 128, fake, 256, None) == 2
    assert lib.arc_silu_mul(fake, 4, 256, 256, -1, fake, 256, None) == 2
    assert lib.arc_silu_mul_quantize_activation(fake, 4, 512, 128, ctypes.byref(prof), fake, fake, None) == 2
    big = arc.ArcProfile(16400, 16, 0x10000, 0x10000, 0)
    assert lib.arc_silu_mul_quantize_activation(fake, 4, 32800, 16400, ctypes.byref(big), fake, fake, None) == 4
    # SwiGLU GEMM: N not a multiple of 32 -> ARC_ERR_SHAPE
    qw = arc.ArcQWeight(48, 256, 320, 16, 0, 0x10000, 0x10000, 0x10000)
    assert lib.arc_gemm_swiglu(fake, fake, fake, 4, ctypes.byref(qw), fake, 24, None, 0, None) == 2
    # MXFP4-ARC: K or S not a multiple of 32 -> ARC_ERR_ALIGN
    assert lib.arc_quantize_activation_mx(fake, 4, 256, ctypes.byref(prof), fake, fake, None) == 3
    prof48 = arc.ArcProfile(272, 32, 0x10000, 0x10000, 0)
    assert lib.arc_quantize_activation_mx(fake, 4, 272, ctypes.byref(prof48), fake, fake, None) == 3
    # the MX tensor offset: largest block scale E8M0_up(amax/6) maps to 2^8
    assert arc.mx_tensor_scale(6.0 * 256) == 1.0
    assert arc.mx_tensor_scale(7.0) == 2.0 ** -(1 - 8)
    assert arc.mx_tensor_scale(0.0) == 1.0
    # gather order for 4-byte channels: still a within-block permutation; bad width refused
    perm = np.random.default_rng(1).permutation(4096).astype(np.int32)
    out = arc.gather_order(perm, 4)
    for b in range(256):
        assert set(out[16 * b:16 * b + 16]) == set(perm[16 * b:16 * b + 16])
    with pytest.raises(arc.ArcError):
        arc.gather_order(perm, 3)
