"""GPU parity of the decode-size paths (M <= 64; Eq.2; north_star decode token
counts M = 1..64): the default arc_linear (quantize kernel + split-K GEMM + fixed-order reduce kernel)
and ARC_LINEAR_FUSED (one kernel: in-kernel quantize + the weight-streaming stream-K GEMM of
stream_gemm.cu, split tiles summed from fp32 partials in a fixed segment order by the last SM).

* Y is within the north_star tolerance 1e-5 * sum|a_i b_i| of the oracle's exact GEMM, recomputed
  by the oracle from the raw bf16 inputs (quantization included), fp32 and bf16 (+ one bf16 ulp);
* every M in 1..64 at one shape; the LLaMA-3-8B site shapes at M = 1, 16, 64;
* repeated calls are bit-identical (fixed reduction order) and leave the workspace's tile
  counters at zero, also under CUDA-graph replay and with one workspace shared by shapes;
* the GEMM called directly (arc_gemm, weights not declared ready) gives the same bits."""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_07475_b200 import synth
from _helpers import dev_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2601_07475_b200 import arc
    assert arc.device_supported()
    return arc


def _problem(A, M, N, K, S, seed=0):
    st = synth.Structure(K, max(S, 16), seed=seed)
    x = synth.activation(M, K, st, seed=seed + 1, device="cuda")
    w = synth.weight(N, K, seed=seed + 2, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=seed + 1000, device="cuda")], s_override=S)
    qw = A.quantize_weight(w, prof)
    return x, w, prof, qw


def _oracle(x, w, prof, qw, rows=None):
    perm, gs, gs_w = prof.perm.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item())
    xb = dev_bits(x) if rows is None else dev_bits(x[torch.as_tensor(rows, device=x.device)])
    ac, asf = oracle.quantize_activation(xb, perm, prof.S, gs)
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, prof.S, gs_w)
    return oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)


def _check(y, yref, bound, bf16):
    tol = bound + (np.abs(yref) * 2.0 ** -8 if bf16 else 0.0)
    err = np.abs(y.float().cpu().numpy().astype(np.float64) - yref)
    assert (err <= tol).all(), f"{(err > tol).sum()} out of tolerance; worst {np.max(err / np.maximum(tol, 1e-300))}"


@pytest.mark.parametrize("M", list(range(1, 65)))
def test_every_decode_m(A, M):
    N, K, S = 384, 1024, 64
    x, w, prof, qw = _problem(A, M, N, K, S, seed=M)
    y = A.linear(x, prof, qw, out_dtype=torch.float32)
    yf = A.linear(x, prof, qw, out_dtype=torch.float32, mode="fused")
    torch.cuda.synchronize()
    ref = _oracle(x, w, prof, qw)
    _check(y, *ref, False)
    _check(yf, *ref, False)


@pytest.mark.parametrize("M", [1, 16, 64])
@pytest.mark.parametrize("site", ["qkv", "o", "gate_up", "down"])
def test_llama3_8b_sites(A, site, M):
    K, N = {n: (k, nn) for n, k, nn in synth.LLAMA3_8B_SITES}[site]
    x, w, prof, qw = _problem(A, M, N, K, 128, seed=K + N + M)
    rows = [0, M - 1] if M > 1 else [0]
    yref, bound = _oracle(x, w, prof, qw, rows)
    for mode in ("auto", "unfused", "fused"):
        y16 = A.linear(x, prof, qw, mode=mode)
        y32 = A.linear(x, prof, qw, out_dtype=torch.float32, mode=mode)
        torch.cuda.synchronize()
        _check(y32[rows], yref, bound, False)
        _check(y16[rows], yref, bound, True)
        assert torch.equal(y16, y32.to(torch.bfloat16))


@pytest.mark.parametrize("M,N,K,S", [(16, 4096, 4096, 128), (3, 130, 2048, 64), (64, 6144, 14336, 128)])
def test_deterministic_and_counters_reset(A, M, N, K, S):
    x, w, prof, qw = _problem(A, M, N, K, S, seed=7)
    ws = A.Workspace("cuda")
    ys = [A.linear(x, prof, qw, out_dtype=torch.float32, ws=ws, mode="fused").clone() for _ in range(4)]
    yd = [A.linear(x, prof, qw, out_dtype=torch.float32, ws=ws, mode="unfused").clone() for _ in range(2)]
    torch.cuda.synchronize()
    assert all(torch.equal(ys[0], y) for y in ys[1:]) and torch.equal(yd[0], yd[1])
    # the GEMM alone gives the two-kernel path's bits
    codes, sf = A.quantize_activation(x, prof)
    y2 = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(yd[0], y2)
    # the GEMM's split-tile counters (u32 [0, 2048) of the linear workspace) and the finished-CTA count
    # (u32 3072) are back at zero; the quantize-ready words and the epoch (u32 2048.., 3073) advance
    cnt = ws.buf[:16384].view(torch.int32)
    assert int(cnt[:2048].count_nonzero().item()) == 0 and int(cnt[3072].item()) == 0
    assert int(cnt[3073].item()) == 4  # four fused launches on this workspace


def test_shared_workspace_across_shapes_and_graph(A):
    """One workspace for several shapes (prefill split-K and decode stream-K) and CUDA-graph replay:
    results stay bit-identical to fresh-workspace calls."""
    probs = [_problem(A, M, N, K, S, seed=M + N) for M, N, K, S in
             [(16, 1024, 4096, 128), (200, 512, 4096, 128), (64, 6144, 4096, 128), (1, 256, 14336, 128)]]
    ref = [A.linear(x, p, q, ws=A.Workspace("cuda"), mode="fused").clone() for x, w, p, q in probs]
    ws = A.Workspace("cuda")
    ws.get(max(A.linear_workspace_size_ex(x.shape[0], q) for x, w, p, q in probs))
    outs = [torch.empty_like(r) for r in ref]
    for _ in range(2):
        for (x, w, p, q), o in zip(probs, outs):
            A.linear(x, p, q, out=o, ws=ws, mode="fused")
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(ref, outs))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for (x, w, p, q), o in zip(probs, outs):
                A.linear(x, p, q, out=o, ws=ws, stream=s, mode="fused")
    for _ in range(3):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(ref, outs))


@pytest.mark.parametrize("M,N,K,S,layout", [(1, 512, 4096, 128, 0), (16, 4096, 4096, 128, 0), (33, 1024, 14336, 128, 1),
                                            (64, 6144, 4096, 64, 0), (7, 300, 1024, 0, 0)])
def test_fused_quantize_phase_bit_exact(A, M, N, K, S, layout):
    """ARC_LINEAR_FUSED quantizes the activation inside the GEMM kernel (one launch): the codes and scales
    it leaves in the workspace are bit-exact against the oracle's quantize_activation, and Y is within
    the GEMM tolerance of the oracle's exact GEMM."""
    st = synth.Structure(K, max(S, 16), seed=K + M)
    x = synth.activation(M, K, st, seed=M + 3, device="cuda")
    w = synth.weight(N, K, seed=N + 4, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=5, device="cuda")], s_override=S, layout=layout)
    qw = A.quantize_weight(w, prof)
    ws = A.Workspace("cuda")
    y_fused = A.linear(x, prof, qw, out_dtype=torch.float32, ws=ws, mode="fused").clone()
    torch.cuda.synchronize()
    Kp = qw.Kp
    code_off = 16384
    sf_off = code_off + (M * (Kp // 2) + 255) // 256 * 256
    codes = ws.buf[code_off:code_off + M * (Kp // 2)].view(M, Kp // 2).cpu().numpy()
    sf = ws.buf[sf_off:sf_off + 128 * (Kp // 16)].cpu().numpy()
    oc, osf = oracle.quantize_activation(dev_bits(x), prof.perm.cpu().numpy(), S, float(prof.gs.item()), layout)
    assert np.array_equal(codes, oc)
    for m in range(M):
        for c in range(Kp // 16):
            o = oracle.sf_offset(m, c, Kp)
            assert sf[o] == osf[o], f"scale byte row {m} block {c}"
    yref, bound = oracle.gemm_reference(oc, osf, *oracle.quantize_weight(dev_bits(w), prof.perm.cpu().numpy(), S,
                                                                          float(qw.gs.item()), layout),
                                        float(prof.gs.item()), float(qw.gs.item()))
    _check(y_fused, yref, bound, False)
