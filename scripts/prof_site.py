"""Run one ARC linear site a few times (for ncu captures): quantize + GEMM.

    python scripts/prof_site.py --site down --M 8192 --iters 3
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--site", default="down")
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--S", type=int, default=128)
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
K, N = {n: (k, nn) for n, k, nn in synth.LLAMA3_8B_SITES}[args.site]
st = synth.Structure(K, args.S, seed=0)
cal = synth.activation(2048, K, st, seed=1000, device="cuda")
prof = A.calibrate([cal], s_override=args.S)
w = synth.weight(N, K, seed=1, device="cuda")
qw = A.quantize_weight(w, prof)
x = synth.activation(args.M, K, st, seed=2, device="cuda")
for _ in range(args.iters):
    codes, sf = A.quantize_activation(x, prof)
    y = A.gemm(codes, sf, prof.gs, qw)
torch.cuda.synchronize()
print("ok", y.shape)
