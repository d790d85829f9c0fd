"""GPU parity of the fused ARC quantization kernel against the oracle (bit-exact).

PAPER.md P:138 (online activation quantization), P:140 (weight duplication),
P:164 (fused kernel), App.D P:591-597 (interleaved layout).  Codes and the
scale bytes of valid rows must equal the oracle's byte for byte.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_07475_b200 import synth
from _helpers import valid_sf_mask, dev_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2601_07475_b200 import arc
    assert arc.device_supported(), "needs sm_100"
    return arc


def _check_act(A, x, perm, S, gs, layout):
    prof = A.profile_from(perm, S, gs, layout)
    codes, sf = A.quantize_activation(x, prof)
    torch.cuda.synchronize()
    oc, osf = oracle.quantize_activation(dev_bits(x), perm, S, gs, layout)
    gc, gsf = codes.cpu().numpy(), sf.cpu().numpy()
    assert np.array_equal(gc, oc), f"codes differ at {np.argwhere(gc != oc)[:5]}"
    mask = valid_sf_mask(x.shape[0], oracle.kp(x.shape[1], S))
    assert np.array_equal(gsf[mask], osf[mask]), "scale bytes differ"


@pytest.mark.parametrize("M,K,S", [(16, 256, 16), (1, 256, 16), (17, 256, 0), (127, 512, 64), (129, 256, 256),
                                   (3, 112, 48), (64, 4096, 128), (5, 14336, 128), (300, 1024, 32)])
@pytest.mark.parametrize("layout", [0, 1])
def test_activation_parity(A, M, K, S, layout):
    st = synth.Structure(K, max(S // 2, 1), seed=M + K)
    x = synth.activation(M, K, st, seed=11, device="cuda")
    perm = synth.random_perm(K, seed=K + S)
    gs = float(np.float32(2688.0) / np.float32(float(x.float().abs().max())))
    _check_act(A, x, perm, S, gs, layout)


def test_activation_parity_calibrated_profile(A):
    """Calibrated perm/S/gs (the online path's real inputs), with saturation: the
    runtime rows exceed the calibration max."""
    K = 2048
    st = synth.Structure(K, 40, seed=0)
    cal = synth.activation(512, K, st, seed=1000, device="cuda")
    prof = A.calibrate([cal])
    assert prof.S_raw == 40 and prof.S == 48
    x = synth.activation(200, K, st, seed=1, device="cuda") * 3
    _check_act(A, x.to(torch.bfloat16), prof.perm.cpu().numpy(), prof.S, float(prof.gs.item()), 0)


def test_adversarial_values(A):
    """E2M1 midpoints, +-0, subnormal-scale blocks, saturating gs, huge values."""
    K, S = 256, 64
    rng = np.random.default_rng(3)
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0], np.float32)
    rows = []
    rows.append(np.tile(np.concatenate([mids, -mids]), K // 16))                  # exact midpoints at gs=1
    rows.append(np.zeros(K, np.float32))                                           # all zero
    rows.append(-np.zeros(K, np.float32))                                          # all -0
    rows.append((rng.standard_normal(K) * 1e-6).astype(np.float32))                # E4M3-subnormal scales
    rows.append((rng.standard_normal(K) * 3e4).astype(np.float32))                 # saturating scales
    r = rng.standard_normal(K).astype(np.float32)
    r[::16] = 0
    r[5::16] = -0.0
    rows.append(r)
    x = torch.tensor(np.stack(rows)).to(torch.bfloat16).cuda()
    for gs in (1.0, 0.37, 448.0 * 6 / 0.5):
        for layout in (0, 1):
            _check_act(A, x, np.arange(K, dtype=np.int32), S, gs, layout)


@pytest.mark.parametrize("N,K,S", [(256, 256, 16), (130, 512, 64), (40, 112, 48), (4096, 4096, 128)])
@pytest.mark.parametrize("layout", [0, 1])
def test_weight_parity(A, N, K, S, layout):
    w = synth.weight(N, K, seed=N, device="cuda")
    perm = synth.random_perm(K, seed=K)
    prof = A.profile_from(perm, S, 1.0, layout)
    qw = A.quantize_weight(w, prof)
    torch.cuda.synchronize()
    gs_w = float(qw.gs.item())
    assert gs_w == oracle.tensor_scale(float(w.float().abs().max()))
    oc, osf = oracle.quantize_weight(dev_bits(w), perm, S, gs_w, layout)
    assert np.array_equal(qw.codes.cpu().numpy(), oc)
    mask = valid_sf_mask(N, qw.Kp)
    assert np.array_equal(qw.sf.cpu().numpy()[mask], osf[mask])


def test_full_size_sampled_rows(A):
    """BASELINE config-2 size (M=8192, down_proj K=14336, S=128) in the bench's launch
    configuration; the oracle recomputes a sample of rows one by one."""
    M, K, S = 8192, 14336, 128
    st = synth.Structure(K, S, seed=0)
    x = synth.activation(M, K, st, seed=5, device="cuda")
    cal = synth.activation(1024, K, st, seed=1000, device="cuda")
    prof = A.calibrate([cal], s_override=S)
    codes, sf = A.quantize_activation(x, prof)
    torch.cuda.synchronize()
    gc, gsf = codes.cpu().numpy(), sf.cpu().numpy()
    perm = prof.perm.cpu().numpy()
    gs = float(prof.gs.item())
    Kp = oracle.kp(K, S)
    # every row: the oracle (OpenMP build, identical per-element arithmetic) quantizes the whole tensor
    with oracle.openmp():
        oc, osf = oracle.quantize_activation(dev_bits(x), perm, S, gs, 0)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gsf[valid_sf_mask(M, Kp)], osf[valid_sf_mask(M, Kp)])


def test_calib_absmax_and_tensor_scale(A):
    x = synth.activation(1000, 512, synth.Structure(512, 8, 0), seed=2, device="cuda")
    cm = A.calib_absmax(x[:600])
    cm = A.calib_absmax(x[600:], cm)
    gs = A.tensor_scale(x)
    torch.cuda.synchronize()
    ocm = oracle.calib_absmax(dev_bits(x))
    assert np.array_equal(cm.cpu().numpy(), ocm)
    assert float(gs.item()) == oracle.tensor_scale(float(ocm.max()))
    z = torch.zeros(4, 64, dtype=torch.bfloat16, device="cuda")
    assert float(A.tensor_scale(z).item()) == 1.0


def test_empty_batch_is_noop(A):
    prof = A.profile_from(np.arange(256, dtype=np.int32), 16, 1.0)
    x = torch.empty(0, 256, dtype=torch.bfloat16, device="cuda")
    codes, sf = A.quantize_activation(x, prof)
    assert codes.shape == (0, 160)


@pytest.mark.parametrize("K,S", [(18944, 64), (17408, 0)])
def test_odd_scale_units_with_one_row_tiles(K, S):
    """Regression: one-row tiles (R = 1) with an odd number of 64-column scale units (Kp/64) used to
    leave the kernel's mbarriers 4-byte aligned (misaligned-address fault); activation and weight
    quantization at such shapes are bit-exact."""
    from paper_2601_07475_b200 import arc as A
    M, N = 37, 96
    st = synth.Structure(K, max(S, 16), seed=K)
    x = synth.activation(M, K, st, seed=1, device="cuda")
    w = synth.weight(N, K, seed=2, device="cuda")
    prof = A.calibrate([synth.activation(128, K, st, seed=3, device="cuda")], s_override=S)
    codes, sf = A.quantize_activation(x, prof)
    qw = A.quantize_weight(w, prof)
    torch.cuda.synchronize()
    perm, gs = prof.perm.cpu().numpy(), float(prof.gs.item())
    oc, osf = oracle.quantize_activation(dev_bits(x), perm, S, gs)
    assert np.array_equal(codes.cpu().numpy(), oc)
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, S, float(qw.gs.item()))
    assert np.array_equal(qw.codes.cpu().numpy(), bc)
