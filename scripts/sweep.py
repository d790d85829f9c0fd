"""Config 3 / config 5 sweeps (BASELINE.json configs[2], configs[4]) -> JSON on stdout.

* S sweep (Fig.8a analogue, "strictly linear correlation with S"): Qwen2.5-7B
  and Qwen2.5-32B linear shapes at M=2048 tokens, S in {0, 64, 128, 256, 512, 1024}: GEMM and
  quantize time, TFLOPS over K+S, overhead vs S=0, linear fit of GEMM time in S.
* Layer-linears comparison (config 5 analogue, linears only): LLaMA-3-8B's four sites at
  M=32768 tokens: ARC (S=128) vs plain NVFP4 (S=0, same kernels) vs BF16 cuBLAS (torch.matmul).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402


def graph_time(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return sorted(ts)[2] * 1e-3


def arc_site(M, K, N, S, seed=0):
    st = synth.Structure(K, max(S, 16), seed=seed)
    prof = A.calibrate([synth.activation(2048, K, st, seed=1000 + seed, device="cuda")], s_override=S)
    qw = A.quantize_weight(synth.weight(N, K, seed=seed + 1, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=seed + 2, device="cuda")
    codes, sf = A.quantize_activation(x, prof)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ws = A.Workspace("cuda")
    tq = graph_time(lambda: A.quantize_activation(x, prof, codes, sf))
    tg = graph_time(lambda: A.gemm(codes, sf, prof.gs, qw, out=y, ws=ws))
    return tq, tg


out = {"s_sweep": [], "layer_linears": {}}
shapes = {"qwen2.5-7b": [("qkv", 3584, 4608), ("o", 3584, 3584), ("gate_up", 3584, 37888), ("down", 18944, 3584)],
          "qwen2.5-32b": [("qkv", 5120, 7168), ("o", 5120, 5120), ("gate_up", 5120, 55296), ("down", 27648, 5120)]}
M = 2048
for model, sites in shapes.items():
    for site, K, N in sites:
        rows = []
        for S in (0, 64, 128, 256, 512, 1024):
            if S > K:
                continue
            tq, tg = arc_site(M, K, N, S)
            rows.append({"S": S, "gemm_us": tg * 1e6, "gemm_tflops": 2.0 * M * N * (K + S) / tg / 1e12,
                         "quant_us": tq * 1e6})
        base = rows[0]["gemm_us"]
        for r in rows:
            r["gemm_overhead_vs_S0"] = r["gemm_us"] / base - 1.0
        Ss = np.array([r["S"] for r in rows], float)
        ts = np.array([r["gemm_us"] for r in rows])
        slope, icpt = np.polyfit(Ss, ts, 1)
        pred = slope * Ss + icpt
        r2 = 1 - np.sum((ts - pred) ** 2) / np.sum((ts - ts.mean()) ** 2)
        out["s_sweep"].append({"model": model, "site": site, "M": M, "K": K, "N": N, "rows": rows,
                               "linear_fit_us_per_channel": slope, "linear_fit_r2": r2})
        print(model, site, [round(r["gemm_us"], 1) for r in rows], "r2=%.4f" % r2, file=sys.stderr)

# config 5 analogue: the 4 LLaMA-3-8B sites at M = 16 x 2048 tokens
M = 32768
tot = {"arc_s128": 0.0, "nvfp4_s0": 0.0, "bf16_cublas": 0.0, "arc_quant_only": 0.0}
for site, K, N in synth.LLAMA3_8B_SITES:
    tq, tg = arc_site(M, K, N, 128)
    tq0, tg0 = arc_site(M, K, N, 0)
    xb = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    wb = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    tb = graph_time(lambda: torch.matmul(xb, wb.t(), out=yb), reps=2)
    del xb, wb, yb
    tot["arc_s128"] += tq + tg
    tot["arc_quant_only"] += tq
    tot["nvfp4_s0"] += tq0 + tg0
    tot["bf16_cublas"] += tb
    out["layer_linears"][site] = {"arc_us": (tq + tg) * 1e6, "arc_quant_us": tq * 1e6, "nvfp4_us": (tq0 + tg0) * 1e6,
                                  "bf16_us": tb * 1e6}
    print(site, out["layer_linears"][site], file=sys.stderr)
out["layer_linears"]["total_us"] = {k: v * 1e6 for k, v in tot.items()}
out["layer_linears"]["arc_vs_nvfp4_overhead"] = tot["arc_s128"] / tot["nvfp4_s0"] - 1.0
out["layer_linears"]["arc_speedup_vs_bf16"] = tot["bf16_cublas"] / tot["arc_s128"]
out["layer_linears"]["M_tokens"] = M
print(json.dumps(out, indent=1))
