"""Time the MLP half of a LLaMA-3-8B layer at prefill M (CUDA graph, CUDA events):
  A: gate_up GEMM (bf16 y) -> fused SiLU-mul+quantize (arc_silu_mul_quantize_activation) -> down GEMM
  B: gate_up GEMM with the SwiGLU epilogue (h) -> plain quantize of h -> down GEMM
and each kernel alone."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H, I, S = 4096, 14336, 128
st = synth.Structure(H, S, seed=0)
sth = synth.Structure(I, S, seed=1)
x = synth.activation(M, H, st, seed=2, device="cuda")
prof1 = A.calibrate([synth.activation(1024, H, st, seed=3, device="cuda")], s_override=S)
wg, wu = synth.weight(I, H, seed=4, device="cuda"), synth.weight(I, H, seed=5, device="cuda")
qgu = A.quantize_weight(torch.cat([wg, wu]), prof1)
qgu_i = A.quantize_weight(A.interleave_gate_up(wg, wu), prof1)
prof2 = A.calibrate([A.silu_mul(synth.gate_up(1024, I, sth, seed=6, device="cuda"))], s_override=S)
qd = A.quantize_weight(synth.weight(H, I, seed=7, device="cuda"), prof2)
c1, s1 = A.quantize_activation(x, prof1)
gu = torch.empty(M, 2 * I, dtype=torch.bfloat16, device="cuda")
h = torch.empty(M, I, dtype=torch.bfloat16, device="cuda")
c2, s2 = A.quantize_activation(h, prof2)
y = torch.empty(M, H, dtype=torch.bfloat16, device="cuda")


def timed(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    return sorted(ts)[2]


parts = {
    "gate_up GEMM (bf16 y)": lambda: A.gemm(c1, s1, prof1.gs, qgu, out=gu),
    "gate_up GEMM + SwiGLU epilogue (h)": lambda: A.gemm_swiglu(c1, s1, prof1.gs, qgu_i, out=h),
    "SiLU-mul + quantize (fused, reads gu)": lambda: A.silu_mul_quantize_activation(gu, prof2, codes=c2, sf=s2),
    "quantize h (K=14336)": lambda: A.quantize_activation(h, prof2, c2, s2),
    "down GEMM": lambda: A.gemm(c2, s2, prof2.gs, qd, out=y),
}
for k, f in parts.items():
    print(f"{k:45s} {timed(f):8.1f} us")


def chain_a():
    A.gemm(c1, s1, prof1.gs, qgu, out=gu)
    A.silu_mul_quantize_activation(gu, prof2, codes=c2, sf=s2)
    A.gemm(c2, s2, prof2.gs, qd, out=y)


def chain_b():
    A.gemm_swiglu(c1, s1, prof1.gs, qgu_i, out=h)
    A.quantize_activation(h, prof2, c2, s2)
    A.gemm(c2, s2, prof2.gs, qd, out=y)


print(f"{'chain A: GEMM -> SiLU-mul+quant -> GEMM':45s} {timed(chain_a, 5):8.1f} us")
print(f"{'chain B: GEMM+SwiGLU -> quant -> GEMM':45s} {timed(chain_b, 5):8.1f} us")
