"""GPU parity of the round-2 decode-size kernels (M <= 64; Eq.1-2):

* arc_quant_small_kernel (direct-gather quantize, taken at M <= 64; x gathered from L2, or from the CTA's
  rows staged in shared memory -- both variants forced in subprocesses): codes and scale bytes bit-exact
  against the oracle's quantize_activation for every M in 1..64 at shapes with residual blocks, K
  padding, S = 0 and both block layouts; and bit-identical to the rows of an M > 64 call of the same
  activation (the staging-ring kernel) -- quantization is row-independent;
* arc_decode_gemm_kernel (cluster split-K, K partials summed in distributed shared memory): Y within
  the north_star tolerance 1e-5 * sum|a_i b_i| of the oracle's exact GEMM of the same quantized
  operands, at shapes covering every cluster size the planner picks (1..8 CTAs), ragged N (not a
  multiple of 128, of 8), half 256-K blocks, fp32 and bf16 output, a row stride ldy > N; repeated
  calls bit-identical (fixed reduction order)."""
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


def _sf_rows_equal(got, want, rows, Kp):
    for m in range(rows):
        for c in range(Kp // 16):
            o = oracle.sf_offset(m, c, Kp)
            if got[o] != want[o]:
                return False, (m, c)
    return True, None


@pytest.mark.parametrize("K,S,layout", [(4096, 128, 0), (1024, 64, 1), (272, 16, 0), (512, 0, 0), (1040, 48, 1),
                                             (14336, 128, 0)])  # long rows: 1024-thread staged CTAs at M >= 32
def test_small_quantize_bit_exact_every_m(A, K, S, layout):
    st = synth.Structure(K, max(S, 16), seed=K + S)
    prof = A.calibrate([synth.activation(256, K, st, seed=11, device="cuda")], s_override=S, layout=layout)
    xbig = synth.activation(200, K, st, seed=12, device="cuda")
    cbig, sfbig = A.quantize_activation(xbig, prof)  # M > 64: the staging-ring kernel
    perm, gs = prof.perm.cpu().numpy(), float(prof.gs.item())
    Kp = oracle.kp(K, S)
    for M in list(range(1, 17)) + [31, 32, 33, 48, 63, 64]:
        c, sf = A.quantize_activation(xbig[:M].contiguous(), prof)
        torch.cuda.synchronize()
        assert torch.equal(c, cbig[:M]), f"M={M}: codes differ from the ring kernel's rows"
        ok, where = _sf_rows_equal(sf.cpu().numpy(), sfbig.cpu().numpy(), M, Kp)
        assert ok, f"M={M}: scale byte {where} differs from the ring kernel's"
        if M in (1, 7, 16, 33, 64):
            oc, osf = oracle.quantize_activation(dev_bits(xbig[:M]), perm, prof.S, gs, layout)
            assert np.array_equal(c.cpu().numpy(), oc), f"M={M}: codes differ from the oracle"
            ok, where = _sf_rows_equal(sf.cpu().numpy(), osf, M, Kp)
            assert ok, f"M={M}: scale byte {where} differs from the oracle"


@pytest.mark.parametrize("M,N,K,S", [
    (1, 384, 1024, 64),       # few K blocks: small clusters
    (16, 4096, 4096, 128),    # LLaMA-3-8B o: clusters of 8, half last K block
    (5, 1000, 4096, 128),     # N % 128 != 0
    (13, 300, 2048, 32),      # N % 8 != 0 -> per-element store of the tail tile
    (64, 2048, 14336, 128),   # long K, M = 64 (N = 64 MMA)
    (33, 20000, 512, 16),     # many tiles: one CTA per tile, no reduction
    (2, 128, 256, 16),        # one tile, one K block
])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_decode_gemm_vs_oracle(A, M, N, K, S, out_dtype):
    st = synth.Structure(K, max(S, 16), seed=N + K)
    x = synth.activation(M, K, st, seed=M + 1, device="cuda")
    w = synth.weight(N, K, seed=N + 2, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=3, device="cuda")], s_override=S)
    qw = A.quantize_weight(w, prof)
    codes, sf = A.quantize_activation(x, prof)
    ldy = (N + 7) // 8 * 8 + 16
    ybuf = torch.full((M, ldy), float("nan"), dtype=out_dtype, device="cuda")
    y = A.gemm(codes, sf, prof.gs, qw, out=ybuf[:, :N])
    y2 = A.gemm(codes, sf, prof.gs, qw, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert torch.equal(y, y2), "repeated decode GEMMs differ (fixed-order reduction)"
    assert torch.isnan(ybuf[:, N:].float()).all(), "wrote past N into the row padding"
    rows = sorted({0, M // 2, M - 1})
    gs, gs_w = float(prof.gs.item()), float(qw.gs.item())
    perm = prof.perm.cpu().numpy()
    ac, asf = oracle.quantize_activation(dev_bits(x[torch.as_tensor(rows, device="cuda")]), perm, prof.S, gs)
    bc, bsf = oracle.quantize_weight(dev_bits(w), perm, prof.S, gs_w)
    yref, bound = oracle.gemm_reference(ac, asf, bc, bsf, gs, gs_w)
    got = y[rows].float().cpu().numpy().astype(np.float64)
    tol = bound + (np.abs(yref) * 2.0 ** -8 if out_dtype == torch.bfloat16 else 0.0)
    err = np.abs(got - yref)
    assert (err <= tol).all(), f"{(err > tol).sum()} outputs out of tolerance; worst {np.max(err / tol)}"


@pytest.mark.parametrize("stage", ["0", "1"])
def test_small_quantize_forced_variants(stage):
    """Both gather variants of arc_quant_small_kernel at every M of the bit-exact test (auto stages the rows
    in shared memory only at M >= 32 with compact rows): ARC_QSMALL_STAGE=0 gathers from L2 everywhere, =1
    stages everywhere (K = 4096 and K = 1040 rows included), in a fresh process (read once per process)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_decode_cluster.py"), "-q", "-x",
                        "-k", "small_quantize_bit_exact"],
                       env={**os.environ, "ARC_QSMALL_STAGE": stage}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
