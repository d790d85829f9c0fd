"""GPU parity of the augmented NVFP4 GEMM (tcgen05.mma kind::mxf4nvf4) against the
oracle's exact integer GEMM: |y - y_ref| <= 1e-5 * sum|a_i b_i| per element
(BASELINE.json north_star tolerance; fp32 accumulation order), plus one bf16 ulp
for bf16 output.  PAPER.md Eq.2."""
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


def _problem(A, M, N, K, S, layout=0, seed=0, S_inj=None):
    st = synth.Structure(K, S if S_inj is None else S_inj, seed=seed)
    x = synth.activation(M, K, st, seed=seed + 1, device="cuda")
    w = synth.weight(N, K, seed=seed + 2, device="cuda")
    cal = synth.activation(max(M, 256), K, st, seed=seed + 1000, device="cuda")
    prof = A.calibrate([cal], s_override=S, layout=layout)
    qw = A.quantize_weight(w, prof)
    return x, w, prof, qw


def _check(y, yref, bound, bf16):
    tol = bound.copy()
    if bf16:
        tol += np.abs(yref) * 2.0 ** -8
    err = np.abs(y - yref)
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} elements out of tolerance; worst err/tol {np.max(err / np.maximum(tol, 1e-300))}"


@pytest.mark.parametrize("M,N,K,S", [(16, 256, 256, 16), (1, 256, 256, 16), (128, 256, 256, 0), (200, 300, 512, 64),
                                     (129, 520, 1024, 128), (64, 64, 112, 48), (257, 1024, 4096, 128),
                                     (520, 600, 1024, 64), (1024, 768, 2048, 128)])
@pytest.mark.parametrize("layout", [0, 1])
def test_gemm_parity_fp32(A, M, N, K, S, layout):
    x, w, prof, qw = _problem(A, M, N, K, S, layout, seed=M + N)
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                        qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()))
    _check(y.cpu().numpy().astype(np.float64), yref, bound, False)


def test_linear_bf16_cfg1(A):
    """Config 1 (M=16, K=256, N=256, S=16) end to end through arc_linear, bf16 out;
    the oracle recomputes quantization AND the GEMM from the raw inputs."""
    M, N, K, S = 16, 256, 256, 16
    x, w, prof, qw = _problem(A, M, N, K, S)
    y = A.linear(x, prof, qw, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    perm, gs, gs_w = prof.perm.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item())
    ac, asf = oracle.quantize_activation(dev_bits(x), perm, S, gs)
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, S, gs_w)
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
    _check(y.float().cpu().numpy().astype(np.float64), yref, bound, True)


def test_same_sign_accumulation(A):
    """Same-sign data at K+S = 14464 stresses the fp32 accumulation (SURVEY hard part 8)."""
    M, N, K, S = 128, 256, 14336, 128
    x = (synth.activation(M, K, synth.Structure(K, S, 0), seed=3, device="cuda").float().abs()).to(torch.bfloat16)
    w = (synth.weight(N, K, seed=4, device="cuda").float().abs()).to(torch.bfloat16)
    prof = A.calibrate([x], s_override=S)
    qw = A.quantize_weight(w, prof)
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                        qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()))
    _check(y.cpu().numpy().astype(np.float64), yref, bound, False)


def test_full_size_sampled_rows(A):
    """BASELINE config-2 prefill size (M=8192, gate-up N=28672? -> qkv N=6144, K=4096,
    S=128) in the bench's launch configuration; the oracle's exact GEMM on sampled rows."""
    M, N, K, S = 8192, 6144, 4096, 128
    x, w, prof, qw = _problem(A, M, N, K, S, seed=7)
    y = A.linear(x, prof, qw, out_dtype=torch.bfloat16)
    codes, sf = A.quantize_activation(x, prof)
    torch.cuda.synchronize()
    # 64 rows: both ends of every 1024-row band, 128-row tile edges and seeded random rows
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([[0, 1, 127, 128, 255, 256, 4095, 4096, 8063, 8064, 8190, 8191],
                                     rng.choice(M, 52, replace=False)])).astype(np.int64)
    with oracle.openmp():
        yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                            qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()), rows=rows)
    _check(y[torch.from_numpy(rows).cuda()].float().cpu().numpy().astype(np.float64), yref, bound, True)


@pytest.mark.parametrize("site", ["qkv", "o", "gate_up", "down"])
def test_bench_sites_full_size(A, site):
    """Every site of bench.py's step at its full size (M = 8192, S = 128) in the bench's launch
    configuration: the whole quantized activation bit-exact against the oracle, the GEMM on 24 sampled
    rows (all N columns) within the north_star bound."""
    K, N = {n: (k, nn) for n, k, nn in synth.LLAMA3_8B_SITES}[site]
    M, S = 8192, 128
    x, w, prof, qw = _problem(A, M, N, K, S, seed=K + N)
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw)
    torch.cuda.synchronize()
    with oracle.openmp():
        oc, osf = oracle.quantize_activation(dev_bits(x), prof.perm.cpu().numpy(), S, float(prof.gs.item()))
    assert np.array_equal(codes.cpu().numpy(), oc)
    rows = np.unique(np.concatenate([[0, 127, 128, M - 1], np.random.default_rng(K).choice(M, 20, replace=False)]))
    with oracle.openmp():
        yref, bound = oracle.gemm_reference(oc, osf, qw.codes.cpu().numpy(), qw.sf.cpu().numpy(),
                                            float(prof.gs.item()), float(qw.gs.item()), rows=rows.astype(np.int64))
    _check(y[torch.from_numpy(rows).cuda()].float().cpu().numpy().astype(np.float64), yref, bound, True)


@pytest.mark.parametrize("M,N", [(4096, 4096), (2944, 2816)])
def test_multi_tile_sampled_rows(A, M, N):
    """Several output tiles per persistent cluster (accumulator double-buffering, stage-ring
    phase wrap across tiles) with ragged M/N edges; exact oracle GEMM on sampled rows that
    cover every 128-row tile position of a 4-CTA cluster."""
    K, S = 1024, 64
    x, w, prof, qw = _problem(A, M, N, K, S, seed=11)
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.arange(0, M, 97), [M - 1, 127, 128, 255, 256, 383, 384, 511]])).astype(np.int64)
    yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                        qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()), rows=rows)
    _check(y[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64), yref, bound, False)


def test_hostio_matches_device_path(A):
    M, N, K, S = 100, 512, 1024, 64
    x, w, prof, qw = _problem(A, M, N, K, S, seed=9)
    y_dev = A.linear(x, prof, qw, out_dtype=torch.bfloat16)
    xh = x.cpu().pin_memory()
    yh = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    ws = torch.zeros(A.linear_hostio_workspace_size(M, qw), dtype=torch.uint8, device="cuda")
    A.linear_hostio(xh, prof, qw, yh, ws)
    assert torch.equal(yh, y_dev.cpu())


def test_cublaslt_cross_check(A):
    """Third-party check of the operand conventions (nibble order, 128x4 scale
    layout): cuBLASLt's NVFP4 GEMM via torch._scaled_mm on our packed operands."""
    if not hasattr(torch, "float4_e2m1fn_x2"):
        pytest.skip("no fp4 dtype")
    M, N, K, S = 256, 512, 1024, 64
    x, w, prof, qw = _problem(A, M, N, K, S, seed=5)
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    a = codes.view(torch.float4_e2m1fn_x2)
    b = qw.codes.view(torch.float4_e2m1fn_x2)
    try:
        ref = torch._scaled_mm(a, b.t(), scale_a=sf.view(torch.float8_e4m3fn), scale_b=qw.sf.view(torch.float8_e4m3fn),
                               out_dtype=torch.float32)
    except Exception as e:  # cuBLASLt build without NVFP4 support
        pytest.skip(f"torch._scaled_mm NVFP4 unavailable: {e}")
    ref = ref / (prof.gs * qw.gs)
    torch.cuda.synchronize()
    assert torch.allclose(y, ref, rtol=1e-4, atol=1e-3 * float(ref.abs().max()))


@pytest.mark.parametrize("M,N,K,S", [(1, 4096, 4096, 128), (16, 6144, 4096, 128), (64, 1024, 14336, 128),
                                     (16, 300, 1024, 64), (33, 4096, 4096, 0)])
def test_decode_splitk_parity(A, M, N, K, S):
    """Decode-size M takes the split-K plan (fp32 partials + fixed-order reduction);
    fp32 and bf16 outputs against the oracle's exact GEMM."""
    x, w, prof, qw = _problem(A, M, N, K, S, seed=M * 7 + N)
    codes, sf = A.quantize_activation(x, prof)
    y32 = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32)
    y16 = A.linear(x, prof, qw, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(),
                                        qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()))
    _check(y32.cpu().numpy().astype(np.float64), yref, bound, False)
    _check(y16.float().cpu().numpy().astype(np.float64), yref, bound, True)
    if M <= 64 and N >= 1024:
        assert A.gemm_workspace_size(M, qw) > 0, "decode-size M should use the split-K plan"


@pytest.mark.parametrize("env", [{"ARC_GEMM_PAIR": "1", "ARC_GEMM_CLP": "2"}, {"ARC_GEMM_PAIR": "1", "ARC_GEMM_CLP": "4"},
                                 {"ARC_GEMM_CL": "1"}, {"ARC_GEMM_CL": "4"}, {"ARC_GEMM_CL": "8"},
                                 {"ARC_GEMM_RASTER": "1"}, {"ARC_GEMM_RASTER": "0"}, {"ARC_GEMM_STREAM": "1"},
                                 {"ARC_GEMM_EPI": "2"}, {"ARC_GEMM_PREF4": "0"}, {"ARC_GEMM_PREF4": "2"},
                                 {"ARC_GEMM_TAIL64": "0"}, {"ARC_DECODE_PULL": "0"}, {"ARC_GEMM_DECODE": "0"},
                                 {"ARC_DECODE_KSMAX": "8"}],
                         ids=["pair2", "pair4", "cl1", "cl4", "cl8", "raster1", "raster0", "stream", "epi2", "pref4_off",
                              "pref4_2x2", "tail64_off", "decode_push", "decode_splitk", "decode_ks8"])
def test_kernel_variants(env):
    """The non-default GEMM kernels/schedules (2-SM cta_group::2 pairs, 4-CTA clusters with
    multicast B, single-CTA, both tile orders, the preferred-cluster modes, the full-box tail, and the
    decode-size variants: bulk-copy push reduction, the split-K + reduce-kernel path, 8-CTA clusters)
    through the same parity tests, in a fresh process (the selection is read once per process)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_gemm.py"), "-q", "-x",
                        "-k", "parity_fp32 or multi_tile or same_sign"],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("site", ["qkv", "o", "gate_up", "down"])
def test_llama3_70b_sites(A, site):
    """BASELINE configs[3] shapes (LLaMA-3-70B: K = 8192 / 28672, N up to 57344) at M = 2048 through
    arc_linear: the whole quantized activation bit-exact against the oracle, Y on 16 sampled rows within
    the north_star bound (+ one bf16 ulp)."""
    K, N = {n: (k, nn) for n, k, nn in synth.LLAMA3_70B_SITES}[site]
    M, S = 2048, 128
    x, w, prof, qw = _problem(A, M, N, K, S, seed=N + 1)
    y = A.linear(x, prof, qw)
    codes, sf = A.quantize_activation(x, prof)
    torch.cuda.synchronize()
    with oracle.openmp():
        oc, osf = oracle.quantize_activation(dev_bits(x), prof.perm.cpu().numpy(), S, float(prof.gs.item()))
    assert np.array_equal(codes.cpu().numpy(), oc)
    rows = np.unique(np.concatenate([[0, 127, 128, M - 1], np.random.default_rng(N).choice(M, 12, replace=False)]))
    with oracle.openmp():
        yref, bound = oracle.gemm_reference(oc, osf, qw.codes.cpu().numpy(), qw.sf.cpu().numpy(),
                                            float(prof.gs.item()), float(qw.gs.item()), rows=rows.astype(np.int64))
    _check(y[torch.from_numpy(rows).cuda()].float().cpu().numpy().astype(np.float64), yref, bound, True)


@pytest.mark.parametrize("pinned", [True, False])
def test_hostio_pipelined_chunks_and_async(A, pinned):
    """arc_linear_hostio pipelines its rows in 128-multiple chunks (H2D / linear / D2H on three streams):
    Y equals arc_linear applied chunk by chunk (bit-exact) and the whole-batch linear within the GEMM
    tolerance; three async calls with distinct workspaces then one wait give the same bits."""
    M, N, K, S = 3000, 640, 1024, 64
    x, w, prof, qw = _problem(A, M, N, K, S, seed=21)
    mc = ((M + 7) // 8 + 127) // 128 * 128
    y_chunks = torch.cat([A.linear(x[r:r + mc], prof, qw) for r in range(0, M, mc)])
    y_whole = A.linear(x, prof, qw, out_dtype=torch.float32)
    xh = x.cpu().pin_memory() if pinned else x.cpu()
    yh = torch.empty(M, N, dtype=torch.bfloat16)
    if pinned:
        yh = yh.pin_memory()
    ws = torch.zeros(A.linear_hostio_workspace_size(M, qw), dtype=torch.uint8, device="cuda")
    A.linear_hostio(xh, prof, qw, yh, ws)
    torch.cuda.synchronize()
    assert torch.equal(yh, y_chunks.cpu())
    assert torch.allclose(yh.float(), y_whole.cpu(), rtol=2 ** -7, atol=1e-3 * float(y_whole.abs().max()))
    outs = [torch.zeros_like(yh) for _ in range(3)]
    wss = [torch.zeros_like(ws) for _ in range(3)]
    for o, wsi in zip(outs, wss):
        A.linear_hostio(xh, prof, qw, o, wsi, wait=False)
    A.linear_hostio_wait()
    assert all(torch.equal(o, yh) for o in outs)
