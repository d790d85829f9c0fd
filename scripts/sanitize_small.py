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
