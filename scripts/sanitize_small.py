"""Small ARC linear runs for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

for (M, K, N, S) in [(16, 256, 256, 16), (129, 512, 520, 64), (300, 1024, 1024, 128), (16, 4096, 4096, 128)]:
    st = synth.Structure(K, max(S // 2, 1), seed=0)
    prof = A.calibrate([synth.activation(256, K, st, seed=1000, device="cuda")], s_override=S)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=2, device="cuda")
    y = A.linear(x, prof, qw)
    y32 = A.linear(x, prof, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    print("ok", M, K, N, S, float(y32.abs().max()))

# fused producers, SwiGLU epilogue, MXFP4-ARC (small shapes)
for (M, K, S) in [(16, 256, 32), (130, 1024, 64)]:
    st = synth.Structure(K, S, seed=3)
    g = synth.rmsnorm_weight(K, seed=4, device="cuda")
    x = synth.activation(M, K, st, seed=5, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=6, device="cuda")], s_override=S)
    A.rmsnorm_quantize_activation(x, g, 1e-5, prof)
    gu = synth.gate_up(M, K, st, seed=7, device="cuda")
    A.silu_mul_quantize_activation(gu, prof)
    pp = A.calibrate([synth.activation(256, K, st, seed=6, device="cuda")], s_override=S, gather_bytes=4)
    gp = torch.stack([gu[:, :K], gu[:, K:]], dim=2).reshape(M, 2 * K).contiguous()
    A.silu_mul_quantize_activation(gp, pp, up_off=A.GU_PAIRS)
    mprof = A.mx_profile(prof, float(x.float().abs().max()))
    qmx = A.quantize_weight_mx(synth.weight(256, K, seed=8, device="cuda"), prof)
    c, sf = A.quantize_activation_mx(x, mprof)
    A.gemm(c, sf, mprof.gs, qmx)
    qgu = A.quantize_weight(A.interleave_gate_up(synth.weight(256, K, seed=9, device="cuda"),
                                                 synth.weight(256, K, seed=10, device="cuda")), prof)
    c1, s1 = A.quantize_activation(x, prof)
    A.gemm_swiglu(c1, s1, prof.gs, qgu)
    torch.cuda.synchronize()
    print("ok producers/mx/swiglu", M, K, S)

# round 2: decode-size cluster split-K GEMM (pull reduction, ks = 1 and ks > 1), the direct-gather decode quantize,
# the preferred-cluster-4 prefill GEMM (raster 0) and the pipelined host-IO linear
for (M, K, N, S) in [(1, 1024, 384, 64), (13, 2048, 300, 32), (64, 4096, 1024, 128), (4, 512, 20000, 16)]:
    st = synth.Structure(K, max(S, 16), seed=11)
    prof = A.calibrate([synth.activation(256, K, st, seed=12, device="cuda")], s_override=S)
    qw = A.quantize_weight(synth.weight(N, K, seed=13, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=14, device="cuda")
    A.linear(x, prof, qw)
    A.linear(x, prof, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    print("ok decode", M, K, N, S)
for (M, K, N, S) in [(512, 1024, 2048, 64), (1024, 2048, 4096, 128)]:
    st = synth.Structure(K, max(S, 16), seed=15)
    prof = A.calibrate([synth.activation(256, K, st, seed=16, device="cuda")], s_override=S)
    qw = A.quantize_weight(synth.weight(N, K, seed=17, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=18, device="cuda")
    A.linear(x, prof, qw)
    xh = x.cpu().pin_memory()
    yh = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    ws = torch.zeros(A.linear_hostio_workspace_size(M, qw), dtype=torch.uint8, device="cuda")
    A.linear_hostio(xh, prof, qw, yh, ws)
    torch.cuda.synchronize()
    print("ok prefill pref4 / hostio", M, K, N, S)
