"""Decode-size 4-site step (LLaMA-3-8B qkv / o / gate_up / down) as the bench's decode sweep times it:
arc_linear per site, CUDA-graph replay, weights (~128 MB) streamed from HBM every step.  Prints us per
step and the HBM fraction for each M and linear mode; environment variables (ARC_*) select kernel
variants.

    python scripts/decode_step.py [M ...]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("ARC_"))
Ms = [int(a) for a in sys.argv[1:]] or [1, 4, 16, 32, 64]
modes = os.environ.get("MODES", "auto,unfused").split(",")


def time_graph(fn, reps=50, warm=3):
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.synchronize()
    for _ in range(warm):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


sites = []
for name, K, N in synth.LLAMA3_8B_SITES:
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    sites.append((name, K, N, prof, qw))
wbytes = sum(qw.codes.numel() + qw.sf.numel() for *_, qw in sites)

for M in Ms:
    xs = [synth.activation(M, K, synth.Structure(K, 8, seed=5), seed=9, device="cuda") for _, K, *_ in sites]
    ys = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _, _, N, *_ in sites]
    wss = [A.Workspace("cuda") for _ in sites]
    dbytes = wbytes + sum(M * K * 2 + M * N * 2 for _, K, N, *_ in sites)
    for mode in modes:
        def step():
            for (name, K, N, prof, qw), x, y, ws in zip(sites, xs, ys, wss):
                A.linear(x, prof, qw, out=y, ws=ws, mode=mode)
        ms = time_graph(step)
        print(f"[{tag}] M={M:2d} mode={mode:8s} {ms * 1e3:7.1f} us/step  {dbytes / (ms * 1e-3) / 1e9:7.0f} GB/s  "
              f"hbm_frac {dbytes / (ms * 1e-3) / 1e9 / HBM:.3f}", flush=True)
