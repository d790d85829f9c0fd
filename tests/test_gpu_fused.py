"""GPU parity of the fused decode linear (arc_linear_ex ARC_LINEAR_FUSED, M <= 128): one kernel
that quantizes the activation (the fused kernel of P:164), runs the augmented NVFP4 GEMM
(Eq.2) over a stream-K split and reduces split tiles in a fixed order.

* The quantized activation it leaves in its workspace is bit-exact against the oracle's
  quantize_activation (codes and scales of every valid row).
* Y is within the north_star tolerance 1e-5 * sum|a_i b_i| of the oracle's exact GEMM,
  recomputed by the oracle from the raw bf16 inputs (+ one bf16 ulp for bf16 output).
* Repeated calls are deterministic and leave the workspace's sync words at zero."""
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


def _problem(A, M, N, K, S, layout=0, seed=0):
    st = synth.Structure(K, S, seed=seed)
    x = synth.activation(M, K, st, seed=seed + 1, device="cuda")
    w = synth.weight(N, K, seed=seed + 2, device="cuda")
    cal = synth.activation(256, K, st, seed=seed + 1000, device="cuda")
    prof = A.calibrate([cal], s_override=S, layout=layout)
    qw = A.quantize_weight(w, prof)
    return x, w, prof, qw


def _oracle(x, w, prof, qw):
    perm, gs, gs_w = prof.perm.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item())
    ac, asf = oracle.quantize_activation(dev_bits(x), perm, prof.S, gs, prof.layout)
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, prof.S, gs_w, prof.layout)
    assert np.array_equal(qw.codes.cpu().numpy(), bc) and np.array_equal(qw.sf.cpu().numpy()[valid_sf_mask(qw.N, qw.Kp)],
                                                                          bsf[valid_sf_mask(qw.N, qw.Kp)])
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
    return ac, asf, yref, bound


def _check(y, yref, bound, bf16):
    tol = bound.copy()
    if bf16:
        tol += np.abs(yref) * 2.0 ** -8
    err = np.abs(y - yref)
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} elements out of tolerance; worst err/tol {np.max(err / np.maximum(tol, 1e-300))}"


def _ws_operand(A, ws, M, qw):
    co, so = A.fused_operand_offsets(M, qw)
    buf = ws.buf
    codes = buf[co:co + M * (qw.Kp // 2)].view(M, qw.Kp // 2).cpu().numpy()
    sf = buf[so:so + 128 * (qw.Kp // 16)].cpu().numpy()
    return codes, sf


# shapes: cfg1; single token; ragged N; S = 0 (plain NVFP4); K not a multiple of the 256-element
# K block (Kp = 1088, 4224); several N tiles per CTA and several CTAs per tile; the full 128-row tile
@pytest.mark.parametrize("M,N,K,S", [(16, 256, 256, 16), (1, 4096, 4096, 128), (16, 6144, 4096, 128),
                                     (64, 1024, 14336, 128), (16, 300, 1024, 64), (33, 4096, 4096, 0),
                                     (100, 520, 1024, 48), (128, 2048, 2048, 256), (7, 64, 112, 48)])
@pytest.mark.parametrize("layout", [0, 1])
def test_fused_linear_parity(A, M, N, K, S, layout):
    x, w, prof, qw = _problem(A, M, N, K, S, layout, seed=M * 13 + N + layout)
    ws = A.Workspace("cuda")
    y32 = A.linear(x, prof, qw, out_dtype=torch.float32, ws=ws, mode="fused")
    torch.cuda.synchronize()
    codes, sf = _ws_operand(A, ws, M, qw)
    ac, asf, yref, bound = _oracle(x, w, prof, qw)
    # the quantized activation, bit-exact (valid rows of the 128-row scale tile)
    assert np.array_equal(codes, ac), "fused quantize: codes differ from the oracle"
    mask = valid_sf_mask(M, qw.Kp)
    assert np.array_equal(sf[mask], asf[mask]), "fused quantize: scales differ from the oracle"
    _check(y32.cpu().numpy().astype(np.float64), yref, bound, False)
    y16 = A.linear(x, prof, qw, out_dtype=torch.bfloat16, ws=ws, mode="fused")
    torch.cuda.synchronize()
    _check(y16.float().cpu().numpy().astype(np.float64), yref, bound, True)
    # the grid-barrier count is back at zero
    assert int(ws.buf[:4].view(torch.int32)[0].item()) == 0


def test_fused_deterministic_and_reusable(A):
    """Same inputs -> bit-identical Y across calls (fixed-order reduction); the workspace is
    shared with an unfused large-M call in between and the fused path still works."""
    M, N, K, S = 16, 6144, 4096, 128
    x, w, prof, qw = _problem(A, M, N, K, S, seed=3)
    ws = A.Workspace("cuda")
    ys = [A.linear(x, prof, qw, out_dtype=torch.float32, ws=ws, mode="fused").clone() for _ in range(3)]
    xb = synth.activation(512, K, synth.Structure(K, S, 3), seed=9, device="cuda")
    A.linear(xb, prof, qw, ws=ws, mode="unfused")
    ys.append(A.linear(x, prof, qw, out_dtype=torch.float32, ws=ws, mode="fused").clone())
    torch.cuda.synchronize()
    for y in ys[1:]:
        assert torch.equal(y, ys[0])


def test_fused_cuda_graph_chain(A):
    """The bench's decode step: the four LLaMA-3-8B sites back to back (PDL between them) in
    one CUDA graph, replayed, all sharing ONE workspace (different N, K -> different split-tile
    counter and operand placements); equal to eager calls and within tolerance of the oracle."""
    M, S = 16, 128
    sites = []
    for i, (name, K, N) in enumerate(synth.LLAMA3_8B_SITES):
        x, w, prof, qw = _problem(A, M, N, K, S, seed=20 + i)
        sites.append((x, w, prof, qw, torch.empty(M, N, dtype=torch.bfloat16, device="cuda")))
    ws = A.Workspace("cuda")
    eager = [A.linear(x, p, q, ws=ws, mode="fused").clone() for x, w, p, q, _ in sites]
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for x, w, p, q, y in sites:  # warm the workspace size
            A.linear(x, p, q, out=y, ws=ws, mode="fused")
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for x, w, p, q, y in sites:
                A.linear(x, p, q, out=y, ws=ws, mode="fused")
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for (x, w, p, q, y), ye in zip(sites, eager):
        assert torch.equal(y, ye)
    x, w, p, q, y = sites[0]
    _, _, yref, bound = _oracle(x, w, p, q)
    _check(y.float().cpu().numpy().astype(np.float64), yref, bound, True)


@pytest.mark.parametrize("min_units", ["1", "4"])
def test_fused_partition_variants(min_units):
    """Other stream-K partitions (fewer CTAs, longer segments) through the parity test, in a
    fresh process (the knob is read once per process)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_fused.py"), "-q", "-x",
                        "-k", "parity and (6144 or 14336 or 520)"],
                       env={**os.environ, "ARC_FUSED_MIN_UNITS": min_units}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_fused_rejects_large_m(A):
    M, N, K, S = 129, 256, 256, 16
    x, w, prof, qw = _problem(A, M, N, K, S)
    with pytest.raises(A.ArcError) as e:
        A.linear(x, prof, qw, mode="fused")
    assert e.value.status == 2
