"""Time arc_gemm alone for LLaMA-3-8B sites (CUDA graph of several launches; L2-cold inputs are not
enforced: each site's operands (>= 46 MB) mostly exceed what one launch leaves in L2)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--site", default="all")
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--S", type=int, default=128)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("ARC_"))
sites = synth.LLAMA3_8B_SITES if args.site == "all" else [s for s in synth.LLAMA3_8B_SITES if s[0] == args.site]
for name, K, N in sites:
    st = synth.Structure(K, args.S, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=args.S)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(args.M, K, st, seed=2, device="cuda")
    codes, sf = A.quantize_activation(x, prof)
    y = torch.empty(args.M, N, dtype=torch.bfloat16, device="cuda")
    ws = A.Workspace("cuda")
    for _ in range(3):
        A.gemm(codes, sf, prof.gs, qw, out=y, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(args.reps):
                A.gemm(codes, sf, prof.gs, qw, out=y, ws=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / args.reps)
    t = sorted(ts)[2]
    fl = 2.0 * args.M * N * (K + args.S)
    print(f"[{tag}] {name} M={args.M} N={N} K={K}+{args.S}: {t*1e3:.1f} us  {fl/t/1e9:.0f} TFLOP/s", flush=True)
    del g, x, codes, sf, y, qw
    torch.cuda.empty_cache()
