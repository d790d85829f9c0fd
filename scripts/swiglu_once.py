import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2601_07475_b200 import arc as A, synth
M, H, I, S = 8192, 4096, 14336, 128
st = synth.Structure(H, S, seed=0)
x = synth.activation(M, H, st, seed=2, device="cuda")
prof = A.calibrate([synth.activation(1024, H, st, seed=3, device="cuda")], s_override=S)
wg, wu = synth.weight(I, H, seed=4, device="cuda"), synth.weight(I, H, seed=5, device="cuda")
q = A.quantize_weight(A.interleave_gate_up(wg, wu), prof)
c, s = A.quantize_activation(x, prof)
h = torch.empty(M, I, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    A.gemm_swiglu(c, s, prof.gs, q, out=h)
torch.cuda.synchronize()
