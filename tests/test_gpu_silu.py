"""GPU parity of the SiLU-mul producer of the down-projection input site (Fig.5 P:157;
SiLU op sequence = DESIGN.md reading Q24):

* arc_silu_mul is bit-exact against the oracle's silu_mul for EVERY finite bf16 gate value
  (all 2^16 patterns, each against several up values) and on the synthetic gate_up recipe;
* arc_silu_mul_quantize_activation (SiLU-mul + reorder + primary + residual NVFP4 in one pass)
  is bit-exact against the oracle's quantize_activation of the oracle's silu_mul, in both
  layouts, across the ring configurations (R = 4 / 2 / 1 rows per tile, 28 primary warps, the
  two-blocks-per-lane variant) and with a gate_up buffer whose up half sits at an offset;
* it equals the unfused GPU chain arc_quantize_activation(arc_silu_mul(gu)) bit for bit;
* arc_linear_silu_mul is within the GEMM tolerance of the oracle's exact GEMM."""
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


def test_silu_mul_every_bf16_gate(A):
    b = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    g = b[((b >> 7) & 0xFF) != 0xFF]                      # finite bf16 patterns
    n = g.size
    K = 512
    rows = (n + K - 1) // K
    gate = np.zeros(rows * K, np.uint16)
    gate[:n] = g
    gen = torch.Generator().manual_seed(1)
    for trial in range(3):
        up = (torch.randn(rows, K, generator=gen) * (4.0 ** trial)).to(torch.bfloat16)
        gu_bits = np.concatenate([gate.reshape(rows, K), dev_bits(up)], axis=1)
        gu = torch.from_numpy(gu_bits.astype(np.int16)).view(torch.bfloat16).cuda()
        h = A.silu_mul(gu)
        torch.cuda.synchronize()
        assert np.array_equal(dev_bits(h), oracle.silu_mul(gu_bits))


def test_fused_silu_stage_every_bf16_gate(A):
    """The fused kernel's SiLU stage (table + closed-form tails + block range check), run as the
    quantizing warps run it, equals the oracle's bf16(SiLU(g)) for all finite bf16 g."""
    b = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    g = b[((b >> 7) & 0xFF) != 0xFF]
    got = A.probe_silu(torch.from_numpy(g.view(np.int16)).cuda()).cpu().numpy().view(np.uint16)
    f = oracle.silu_f32(g).view(np.uint32).astype(np.uint64)
    want = ((f + 0x7FFF + ((f >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(got, want), f"{(got != want).sum()} patterns differ"


@pytest.mark.parametrize("M,K", [(1, 16), (37, 256), (64, 4096), (9, 14336)])
def test_silu_mul_recipe(A, M, K):
    st = synth.Structure(K, 16, seed=K)
    gu = synth.gate_up(M, K, st, seed=M + K, device="cuda")
    h = A.silu_mul(gu)
    torch.cuda.synchronize()
    assert np.array_equal(dev_bits(h), oracle.silu_mul(dev_bits(gu)))


# K = 256 (R = 4), 4096 (R = 2), 8192 (R = 2, 32 KB rows), 14336 (R = 1, 28 primary warps),
# 16384 (two blocks per primary lane), ragged M / K
@pytest.mark.parametrize("M,K,S", [(16, 256, 16), (300, 4096, 128), (70, 8192, 64), (77, 14336, 128),
                                   (12, 16384, 256), (130, 1024, 0), (5, 112, 48)])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("pairs", [False, True])
def test_silu_mul_quantize_bit_exact(A, M, K, S, layout, pairs):
    st = synth.Structure(K, max(S, 16), seed=K + S)
    gu = synth.gate_up(M, K, st, seed=M * 3 + K + layout, device="cuda")
    cal = A.silu_mul(synth.gate_up(256, K, st, seed=99, device="cuda"))
    prof = A.calibrate([cal], s_override=S, layout=layout, gather_bytes=4 if pairs else 2)
    if pairs:  # the same gate/up values as (g_j, u_j) adjacent pairs
        gp = torch.stack([gu[:, :K], gu[:, K:]], dim=2).reshape(M, 2 * K).contiguous()
        codes, sf = A.silu_mul_quantize_activation(gp, prof, up_off=A.GU_PAIRS)
        assert torch.equal(A.silu_mul(gp, up_off=A.GU_PAIRS), A.silu_mul(gu))
    else:
        codes, sf = A.silu_mul_quantize_activation(gu, prof)
    c2, s2 = A.quantize_activation(A.silu_mul(gu), prof)
    torch.cuda.synchronize()
    h_or = oracle.silu_mul(dev_bits(gu))
    oc, osf = oracle.quantize_activation(h_or, prof.perm.cpu().numpy(), S, float(prof.gs.item()), layout)
    mask = valid_sf_mask(M, _kp(K, S))
    assert np.array_equal(codes.cpu().numpy(), oc), "fused SiLU-mul+quantize codes differ from the oracle"
    assert np.array_equal(sf.cpu().numpy()[mask], osf[mask]), "fused SiLU-mul+quantize scales differ"
    mt = torch.from_numpy(mask).cuda()
    assert torch.equal(codes, c2) and torch.equal(sf.view(-1)[mt], s2.view(-1)[mt])


def test_silu_mul_quantize_offset_up(A):
    """gate in columns [0, K), 64 pad columns, up in [K + 64, 2K + 64); row stride 2K + 128."""
    M, K, S = 50, 2048, 64
    st = synth.Structure(K, 64, seed=4)
    base = synth.gate_up(M, K, st, seed=8, device="cuda")
    buf = torch.zeros(M, 2 * K + 128, dtype=torch.bfloat16, device="cuda")
    buf[:, :K] = base[:, :K]
    buf[:, K + 64:2 * K + 64] = base[:, K:]
    prof = A.calibrate([A.silu_mul(synth.gate_up(128, K, st, seed=3, device="cuda"))], s_override=S)
    codes, sf = A.silu_mul_quantize_activation(buf, prof, up_off=K + 64)
    torch.cuda.synchronize()
    oc, osf = oracle.quantize_activation(oracle.silu_mul(dev_bits(buf), K=K, up_off=K + 64),
                                         prof.perm.cpu().numpy(), S, float(prof.gs.item()))
    assert np.array_equal(codes.cpu().numpy(), oc)
    mask = valid_sf_mask(M, _kp(K, S))
    assert np.array_equal(sf.cpu().numpy()[mask], osf[mask])


def test_silu_mul_quantize_full_size_sampled_rows(A):
    """The bench's down-proj input site at full prefill size (M = 8192, K = 14336, S = 128),
    bit-exact on sampled rows (the oracle runs row by row)."""
    M, K, S = 8192, 14336, 128
    st = synth.Structure(K, S, seed=21)
    gu = synth.gate_up(M, K, st, seed=22, device="cuda")
    prof = A.calibrate([A.silu_mul(synth.gate_up(1024, K, st, seed=23, device="cuda"))], s_override=S)
    codes, sf = A.silu_mul_quantize_activation(gu, prof)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 31, 32, 127, 128, 129, 4095, 5000, 8191])
    oc, osf = oracle.quantize_activation(oracle.silu_mul(dev_bits(gu[torch.from_numpy(rows).cuda()])),
                                         prof.perm.cpu().numpy(), S, float(prof.gs.item()))
    assert np.array_equal(codes.cpu().numpy()[rows], oc)
    Kp = _kp(K, S)
    sfn = sf.cpu().numpy()
    for i, m in enumerate(rows):
        for c in range(Kp // 16):
            assert sfn[oracle.sf_offset(int(m), c, Kp)] == osf[oracle.sf_offset(i, c, Kp)]


@pytest.mark.parametrize("M,N,K,S", [(16, 256, 256, 16), (200, 600, 4096, 128), (16, 4096, 14336, 128)])
def test_linear_silu_mul_parity(A, M, N, K, S):
    st = synth.Structure(K, S, seed=N)
    gu = synth.gate_up(M, K, st, seed=N + 2, device="cuda")
    w = synth.weight(N, K, seed=N + 1, device="cuda")
    prof = A.calibrate([A.silu_mul(synth.gate_up(256, K, st, seed=5, device="cuda"))], s_override=S)
    qw = A.quantize_weight(w, prof)
    y = A.linear_silu_mul(gu, prof, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    perm, gs, gs_w = prof.perm.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item())
    ac, asf = oracle.quantize_activation(oracle.silu_mul(dev_bits(gu)), perm, S, gs)
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, S, gs_w)
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
    err = np.abs(y.cpu().numpy().astype(np.float64) - yref)
    assert (err <= bound).all(), f"worst err/bound {np.max(err / np.maximum(bound, 1e-300))}"


# ----------------------------------------------------------------------------- SwiGLU GEMM epilogue
@pytest.mark.parametrize("M,I,K,S", [(16, 256, 256, 16), (300, 640, 4096, 128), (1000, 1024, 1024, 64),
                                     (16, 14336, 4096, 128)])
def test_gemm_swiglu_matches_silu_of_gemm(A, M, I, K, S):
    """h from the SwiGLU epilogue == arc_silu_mul of the de-interleaved bf16 arc_gemm output, bit
    for bit (the same kernel computes y; split-K at M = 16), and y over the interleaved weight
    is within the GEMM tolerance of the oracle's exact GEMM (silu_mul itself is pinned
    exhaustively in test_silu_mul_every_bf16_gate)."""
    st = synth.Structure(K, max(S, 16), seed=I)
    x = synth.activation(M, K, st, seed=I + 1, device="cuda")
    wg = synth.weight(I, K, seed=I + 2, device="cuda")
    wu = synth.weight(I, K, seed=I + 3, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=7, device="cuda")], s_override=S)
    qw = A.quantize_weight(A.interleave_gate_up(wg, wu), prof)
    codes, sf = A.quantize_activation(x, prof)
    h = A.gemm_swiglu(codes, sf, prof.gs, qw)
    y = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.bfloat16)
    h2 = A.silu_mul(A.deinterleave_gate_up(y).contiguous())
    torch.cuda.synchronize()
    assert torch.equal(h, h2), f"{(h != h2).sum().item()} of {h.numel()} differ"
    if M * I <= 300 * 640:
        yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                            qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()))
        y32 = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32).cpu().numpy().astype(np.float64)
        assert (np.abs(y32 - yref) <= bound).all()


def test_silu_mul_quantize_odd_scale_units(A):
    """Regression (one-row tiles, odd Kp/64): K = 14336, S = 64 -> Kp/64 = 225."""
    M, K, S = 20, 14336, 64
    st = synth.Structure(K, S, seed=5)
    gu = synth.gate_up(M, K, st, seed=6, device="cuda")
    prof = A.calibrate([A.silu_mul(synth.gate_up(128, K, st, seed=7, device="cuda"))], s_override=S)
    codes, sf = A.silu_mul_quantize_activation(gu, prof)
    torch.cuda.synchronize()
    oc, osf = oracle.quantize_activation(oracle.silu_mul(dev_bits(gu)), prof.perm.cpu().numpy(), S,
                                         float(prof.gs.item()))
    assert np.array_equal(codes.cpu().numpy(), oc)


def _bf16_key(bits: np.ndarray) -> np.ndarray:
    """Order-preserving integer key of bf16 bit patterns (-0 and +0 adjacent)."""
    b = bits.astype(np.int64)
    return np.where(b < 0x8000, b + 0x8000, 0x7FFF - (b & 0x7FFF))


def _bf16_from_key(k: np.ndarray) -> np.ndarray:
    return np.where(k >= 0x8000, k - 0x8000, 0x8000 | (0x7FFF - k)).astype(np.uint16)


def _bf16_bits_rn(v: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(torch.bfloat16).view(torch.int16) \
        .numpy().view(np.uint16)


@pytest.mark.parametrize("M,I,K,S", [(16, 256, 256, 16), (300, 640, 4096, 128), (1000, 1024, 1024, 64),
                                     (16, 14336, 4096, 128), (64, 2048, 14336, 128)])
def test_gemm_swiglu_vs_oracle(A, M, I, K, S):
    """The SwiGLU epilogue against the oracle alone: every h equals oracle.silu_mul(g', u') for some
    bf16 g', u' that round a value inside the GEMM tolerance interval of the oracle's exact gate /
    up outputs (y_ref +- (1e-5 sum|ab| + fp32 rounding of alpha*acc)) -- normally one or both bf16
    neighbours of y_ref.  Elements whose interval spans more than 3 bf16 values (|y| near 0 under
    heavy cancellation) are counted and must be rare."""
    st = synth.Structure(K, max(S, 16), seed=I + 5)
    x = synth.activation(M, K, st, seed=I + 6, device="cuda")
    wg = synth.weight(I, K, seed=I + 7, device="cuda")
    wu = synth.weight(I, K, seed=I + 8, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=8, device="cuda")], s_override=S)
    qw = A.quantize_weight(A.interleave_gate_up(wg, wu), prof)
    codes, sf = A.quantize_activation(x, prof)
    h = dev_bits(A.gemm_swiglu(codes, sf, prof.gs, qw))
    torch.cuda.synchronize()
    perm, gs, gs_w = prof.perm.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item())
    # operands from the oracle (independent of the GPU quantizers)
    ac, asf = oracle.quantize_activation(dev_bits(x), perm, S, gs)
    bc, bsf = oracle.quantize_weight(dev_bits(A.interleave_gate_up(wg, wu)), perm, S, gs_w)
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
    slack = bound + np.abs(yref) * 2.0 ** -23
    lo = _bf16_key(_bf16_bits_rn(yref - slack))
    hi = _bf16_key(_bf16_bits_rn(yref + slack))
    lo, hi = np.minimum(lo, hi), np.maximum(lo, hi)
    v = lambda a: a.reshape(M, I // 16, 2, 16)  # noqa: E731  (interleave layout: 16 gate, 16 up columns)
    glo, ghi, ulo, uhi = v(lo)[:, :, 0].reshape(M, I), v(hi)[:, :, 0].reshape(M, I), \
        v(lo)[:, :, 1].reshape(M, I), v(hi)[:, :, 1].reshape(M, I)
    ok = np.zeros((M, I), bool)
    for dg in range(3):
        for du in range(3):
            g = _bf16_from_key(np.minimum(glo + dg, ghi))
            u = _bf16_from_key(np.minimum(ulo + du, uhi))
            ok |= oracle.silu_mul(np.concatenate([g, u], axis=1)) == h
    wide = ((ghi - glo) > 2) | ((uhi - ulo) > 2)
    bad = ~ok & ~wide
    assert not bad.any(), f"{bad.sum()} of {bad.size} h values match no candidate; first at {np.argwhere(bad)[0]}"
    # wide intervals (|y| small against sum|ab|): every bf16 pair inside them
    unchecked = 0
    for m, i in np.argwhere(wide & ~ok):
        gk = np.arange(glo[m, i], ghi[m, i] + 1)
        uk = np.arange(ulo[m, i], uhi[m, i] + 1)
        if gk.size * uk.size > 1 << 18:
            unchecked += 1
            continue
        G, U = np.meshgrid(gk, uk, indexing="ij")
        cand = oracle.silu_mul(np.concatenate([_bf16_from_key(G.reshape(1, -1)), _bf16_from_key(U.reshape(1, -1))],
                                              axis=1))
        assert (cand == h[m, i]).any(), f"h[{m},{i}] matches no bf16 (g, u) inside the tolerance intervals"
    assert unchecked <= max(1, h.size // 10000), f"{unchecked} intervals too wide to enumerate"
