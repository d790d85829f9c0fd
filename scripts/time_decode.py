"""Decode-size ARC linear latency per LLaMA-3-8B site, fused (one kernel) and unfused
(quantize + split-K GEMM + reduction), CUDA-graph replay (rotating weights so the weight
stream comes from HBM)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

S = 128
MODES = sys.argv[1:] or ["fused", "unfused"]
for M in (1, 16, 64, 128):
  for mode in MODES:
    for site, K, N in synth.LLAMA3_8B_SITES:
        st = synth.Structure(K, S, seed=0)
        prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=S)
        w = synth.weight(N, K, seed=1, device="cuda")
        qws = [A.quantize_weight(w, prof) for _ in range(max(2, int(4 * 126e6 // (N * K * 0.6)) + 1))]
        del w
        x = synth.activation(M, K, st, seed=2, device="cuda")
        y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        ws = A.Workspace("cuda")
        for q in qws[:2]:
            A.linear(x, prof, q, out=y, ws=ws, mode=mode)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for q in qws:
                    A.linear(x, prof, q, out=y, ws=ws, mode=mode)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / len(qws))
        t = sorted(ts)[2] * 1e-3
        wbytes = N * qws[0].Kp * 9 / 16
        tot = wbytes + M * K * 2 + M * N * 2
        print(f"decode {mode:7s} M={M:3d} {site:8s} N={N:6d} K={K:6d}: {t*1e6:7.2f} us  weights {wbytes/1e6:6.1f} MB  "
              f"{tot/t/1e9:6.0f} GB/s  ws {A.linear_workspace_size_ex(M, qws[0], mode)/1e6:.2f} MB")
        del qws
