"""One launch each of arc_gemm (and optionally cuBLASLt NVFP4 on the same operands) for ncu
metric comparison: python scripts/prof_compare.py [--cublas] [--sites qkv,down]."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cublas", action="store_true")
ap.add_argument("--sites", default="qkv,down")
ap.add_argument("--M", type=int, default=8192)
args = ap.parse_args()
for site, K, N in synth.LLAMA3_8B_SITES:
    if site not in args.sites.split(","):
        continue
    S = 128
    st = synth.Structure(K, S, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=S)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(args.M, K, st, seed=2, device="cuda")
    codes, sf = A.quantize_activation(x, prof)
    y = torch.empty(args.M, N, dtype=torch.bfloat16, device="cuda")
    for _ in range(2):
        A.gemm(codes, sf, prof.gs, qw, out=y)
    if args.cublas:
        a = codes.view(torch.float4_e2m1fn_x2)
        b = qw.codes.view(torch.float4_e2m1fn_x2)
        for _ in range(2):
            torch._scaled_mm(a, b.t(), scale_a=sf.view(torch.float8_e4m3fn), scale_b=qw.sf.view(torch.float8_e4m3fn),
                             out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
