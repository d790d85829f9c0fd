"""One launch each of the fused producers at the bench's prefill size (M=8192) for ncu:
RMSNorm+quantize (K=4096), SiLU-mul+quantize (K=14336), gate_up GEMM with the SwiGLU epilogue."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

M, H, I, S = 8192, 4096, 14336, 128
st = synth.Structure(H, S, seed=0)
sti = synth.Structure(I, S, seed=1)
x = synth.activation(M, H, st, seed=2, device="cuda")
g = synth.rmsnorm_weight(H, seed=3, device="cuda")
p1 = A.calibrate([A.rmsnorm(synth.activation(1024, H, st, seed=4, device="cuda"), g, 1e-5)], s_override=S)
gu = synth.gate_up(M, I, sti, seed=5, device="cuda")
p2 = A.calibrate([A.silu_mul(synth.gate_up(1024, I, sti, seed=6, device="cuda"))], s_override=S)
q = A.quantize_weight(A.interleave_gate_up(synth.weight(I, H, seed=7, device="cuda"),
                                           synth.weight(I, H, seed=8, device="cuda")), p1)
c1, s1 = A.rmsnorm_quantize_activation(x, g, 1e-5, p1)
c2, s2 = A.silu_mul_quantize_activation(gu, p2)
h = torch.empty(M, I, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    A.rmsnorm_quantize_activation(x, g, 1e-5, p1, c1, s1)
    A.silu_mul_quantize_activation(gu, p2, codes=c2, sf=s2)
    A.gemm_swiglu(c1, s1, p1.gs, q, out=h)
torch.cuda.synchronize()
