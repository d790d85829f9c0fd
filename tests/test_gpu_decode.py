"""GPU parity of the decode-size path (M <= 64): arc_linear = arc_quantize_activation + the
weight-streaming stream-K GEMM (stream_gemm.cu), whose split tiles are summed from fp32 partials
in a fixed segment order by the last SM to finish them (Eq.2; north_star
decode token counts M = 1..64).

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
    torch.cuda.synchronize()
    _check(y, *_oracle(x, w, prof, qw), False)


@pytest.mark.parametrize("M", [1, 16, 64])
@pytest.mark.parametrize("site", ["qkv", "o", "gate_up", "down"])
def test_llama3_8b_sites(A, site, M):
    K, N = {n: (k, nn) for n, k, nn in synth.LLAMA3_8B_SITES}[site]
    x, w, prof, qw = _problem(A, M, N, K, 128, seed=K + N + M)
    y16 = A.linear(x, prof, qw)
    y32 = A.linear(x, prof, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = [0, M - 1] if M > 1 else [0]
    yref, bound = _oracle(x, w, prof, qw, rows)
    _check(y32[rows], yref, bound, False)
    _check(y16[rows], yref, bound, True)
    assert torch.equal(y16, y32.to(torch.bfloat16))


@pytest.mark.parametrize("M,N,K,S", [(16, 4096, 4096, 128), (3, 130, 2048, 64), (64, 6144, 14336, 128)])
def test_deterministic_and_counters_reset(A, M, N, K, S):
    x, w, prof, qw = _problem(A, M, N, K, S, seed=7)
    ws = A.Workspace("cuda")
    ys = [A.linear(x, prof, qw, out_dtype=torch.float32, ws=ws).clone() for _ in range(4)]
    torch.cuda.synchronize()
    assert all(torch.equal(ys[0], y) for y in ys[1:])
    # the GEMM alone (weights not declared ready: no early weight stream) gives the same bits
    codes, sf = A.quantize_activation(x, prof)
    y2 = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], y2)
    # the GEMM's tile counters (the first 16 KB of the linear workspace) are back at zero
    assert int(ws.buf[:16384].count_nonzero().item()) == 0


def test_shared_workspace_across_shapes_and_graph(A):
    """One workspace for several shapes (prefill split-K and decode stream-K) and CUDA-graph replay:
    results stay bit-identical to fresh-workspace calls."""
    probs = [_problem(A, M, N, K, S, seed=M + N) for M, N, K, S in
             [(16, 1024, 4096, 128), (200, 512, 4096, 128), (64, 6144, 4096, 128), (1, 256, 14336, 128)]]
    ref = [A.linear(x, p, q, ws=A.Workspace("cuda")).clone() for x, w, p, q in probs]
    ws = A.Workspace("cuda")
    ws.get(max(A.linear_workspace_size_ex(x.shape[0], q) for x, w, p, q in probs))
    outs = [torch.empty_like(r) for r in ref]
    for _ in range(2):
        for (x, w, p, q), o in zip(probs, outs):
            A.linear(x, p, q, out=o, ws=ws)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(ref, outs))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for (x, w, p, q), o in zip(probs, outs):
                A.linear(x, p, q, out=o, ws=ws, stream=s)
    for _ in range(3):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(ref, outs))
