"""GPU parity of MXFP4-ARC (reading Q25): arc_quantize_activation_mx /
arc_quantize_weight_mx are bit-exact against the oracle (codes and the scales of every valid row)
in both layouts and across the kernel's ring configurations, and arc_gemm over the MX operands is
within the north_star tolerance of the oracle's exact GEMM (which equals the float64 MX dot
products, tests/test_oracle_mx.py)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_07475_b200 import synth
from _helpers import dev_bits, valid_sf_mask

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2601_07475_b200 import arc
    assert arc.device_supported()
    return arc


def _kp(K, S):
    return (K + S + 63) // 64 * 64


@pytest.mark.parametrize("M,K,S", [(16, 256, 32), (300, 4096, 128), (77, 14336, 128), (130, 1024, 0),
                                   (5, 96, 64), (12, 16384, 256)])
@pytest.mark.parametrize("layout", [0, 1])
def test_mx_quantize_bit_exact(A, M, K, S, layout):
    st = synth.Structure(K, max(S, 32), seed=K + S)
    x = synth.activation(M, K, st, seed=M + K + layout, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=9, device="cuda")], s_override=S, layout=layout)
    mprof = A.mx_profile(prof, float(x.float().abs().max()))
    c = -int(np.log2(float(mprof.gs.item())))
    codes, sf = A.quantize_activation_mx(x, mprof)
    torch.cuda.synchronize()
    oc, osf = oracle.quantize_mx(dev_bits(x), prof.perm.cpu().numpy(), S, c, layout=layout)
    mask = valid_sf_mask(M, _kp(K, S))
    assert np.array_equal(codes.cpu().numpy(), oc)
    assert np.array_equal(sf.cpu().numpy()[mask], osf[mask])


@pytest.mark.parametrize("M,N,K,S", [(16, 256, 256, 32), (200, 600, 4096, 128), (1000, 512, 1024, 64)])
def test_mx_weight_and_gemm(A, M, N, K, S):
    st = synth.Structure(K, max(S, 32), seed=N)
    x = synth.activation(M, K, st, seed=N + 1, device="cuda")
    w = synth.weight(N, K, seed=N + 2, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=3, device="cuda")], s_override=S)
    mprof = A.mx_profile(prof, float(x.float().abs().max()))
    qw = A.quantize_weight_mx(w, prof)
    codes, sf = A.quantize_activation_mx(x, mprof)
    y = A.gemm(codes, sf, mprof.gs, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    perm = prof.perm.cpu().numpy()
    cx, cw = -int(np.log2(float(mprof.gs.item()))), -int(np.log2(float(qw.gs.item())))
    bc, bsf = oracle.quantize_mx(dev_bits(w), perm, S, cw, weight=True)
    assert np.array_equal(qw.codes.cpu().numpy(), bc)
    mask = valid_sf_mask(N, _kp(K, S))
    assert np.array_equal(qw.sf.cpu().numpy()[mask], bsf[mask])
    ac, asf = oracle.quantize_mx(dev_bits(x), perm, S, cx)
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, 2.0 ** -cx, 2.0 ** -cw)
    err = np.abs(y.cpu().numpy().astype(np.float64) - yref)
    assert (err <= bound).all(), f"worst err/bound {np.max(err / np.maximum(bound, 1e-300))}"


@pytest.mark.parametrize("layout", [0, 1])
def test_mx_wide_dynamic_range_bit_exact(A, layout):
    """blocks whose exponent leaves E4M3's powers of two for the tensor offset (dynamic
    range > 2^17, runtime values above the calibrated max) are clamped as reading Q25b says -- codes
    and scales bit-exact against the oracle, activation and weight mode."""
    M, K, S = 64, 1024, 64
    st = synth.Structure(K, S, seed=3)
    x = synth.activation(M, K, st, seed=4, device="cuda").float()
    g = torch.Generator(device="cuda").manual_seed(5)
    x = x * torch.exp2(torch.randint(-24, 9, (1, K), generator=g, device="cuda").float())
    x = x.to(torch.bfloat16)
    prof = A.calibrate([synth.activation(256, K, st, seed=9, device="cuda")], s_override=S, layout=layout)
    mprof = A.mx_profile(prof, prof.M)      # offset from the calibration max, below the runtime max
    c = -int(np.log2(float(mprof.gs.item())))
    codes, sf = A.quantize_activation_mx(x, mprof)
    qw = A.quantize_weight_mx(x[:40].contiguous(), prof)
    torch.cuda.synchronize()
    perm = prof.perm.cpu().numpy()
    oc, osf = oracle.quantize_mx(dev_bits(x), perm, S, c, layout=layout)
    mask = valid_sf_mask(M, _kp(K, S))
    assert np.array_equal(codes.cpu().numpy(), oc)
    assert np.array_equal(sf.cpu().numpy()[mask], osf[mask])
    cw = -int(np.log2(float(qw.gs.item())))
    assert cw == oracle.mx_offset(float(x[:40].float().abs().max()))
    bc, bsf = oracle.quantize_mx(dev_bits(x[:40]), perm, S, cw, weight=True, layout=layout)
    mw = valid_sf_mask(40, _kp(K, S))
    assert np.array_equal(qw.codes.cpu().numpy(), bc)
    assert np.array_equal(qw.sf.cpu().numpy()[mw], bsf[mw])


# ----------------------------------------------------------------------------- native MX format
@pytest.mark.parametrize("M,K,S", [(16, 256, 32), (300, 4096, 128), (77, 14336, 128), (5, 96, 64), (130, 1024, 0)])
@pytest.mark.parametrize("layout", [0, 1])
def test_mx_native_quantize_bit_exact(A, M, K, S, layout):
    """arc_quantize_mx_native (UE8M0 per 32-block, full exponent range) bit-exact against the oracle:
    activations and duplicated weights, both layouts, incl. blocks 2^60 apart (no offset to clamp to)."""
    st = synth.Structure(K, max(S, 32), seed=K + S + 1)
    x = synth.activation(M, K, st, seed=M + K, device="cuda").float()
    x[:, : K // 4] *= 2.0 ** 40
    x[:, K // 4: K // 2] *= 2.0 ** -20
    x = x.to(torch.bfloat16)
    prof = A.calibrate([synth.activation(256, K, st, seed=9, device="cuda")], s_override=S, layout=layout)
    perm = prof.perm.cpu().numpy()
    Km = oracle.kpm(K, S)
    for weight in (False, True):
        codes, sf = A.quantize_mx_native(x, prof, weight=weight)
        torch.cuda.synchronize()
        oc, osf = oracle.quantize_mx_native(dev_bits(x), perm, S, weight=weight, layout=layout)
        assert np.array_equal(codes.cpu().numpy(), oc), weight
        mask = np.zeros(osf.size, bool)
        for r in range(M):
            for b in range(Km // 32):
                mask[oracle.sf_offset(r, b, Km // 2)] = True
        assert np.array_equal(sf.cpu().numpy()[mask], osf[mask]), weight


@pytest.mark.parametrize("M,N,K,S", [(16, 256, 256, 32), (200, 600, 4096, 128), (1000, 512, 1024, 64), (1, 4096, 4096, 128),
                                     (256, 1024, 14336, 128)])
def test_mx_native_gemm(A, M, N, K, S):
    """arc_gemm_mx_native (tcgen05 kind::mxf4 scale_vec::2X, the byte pair of each MMA selected by the SF
    ids) within the north_star bound of the oracle's exact native-MX GEMM; prefill, ragged and split-K."""
    st = synth.Structure(K, max(S, 32), seed=N)
    x = synth.activation(M, K, st, seed=N + 1, device="cuda")
    w = synth.weight(N, K, seed=N + 2, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=3, device="cuda")], s_override=S)
    ac, asf = A.quantize_mx_native(x, prof)
    bc, bsf = A.quantize_mx_native(w, prof, weight=True)
    y = A.gemm_mx_native(ac, asf, bc, bsf, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, M - 1], np.arange(0, M, max(1, M // 16))])).astype(np.int64)
    with oracle.openmp():
        yref, bound = oracle.gemm_mx_native_reference(ac.cpu().numpy(), asf.cpu().numpy(), bc.cpu().numpy(),
                                                      bsf.cpu().numpy(), rows=rows)
    err = np.abs(y.cpu().numpy().astype(np.float64)[rows] - yref)
    assert (err <= bound).all(), f"{(err > bound).sum()} out of tolerance; worst {np.max(err / np.maximum(bound, 1e-300))}"
