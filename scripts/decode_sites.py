"""Decode-size per-site latency of the ARC linear (LLaMA-3-8B sites), HBM-cold weights: each site
rotates over R weight copies (R x weight bytes >= 512 MB, > 4x L2) inside one CUDA graph, so every
call streams its weights from HBM.  Prints quantize alone, GEMM alone and arc_linear per call, with
the weight-streaming bound (weight bytes / measured HBM)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("ARC_"))


def t(fn, n):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(n):
                fn(i)
    torch.cuda.synchronize()
    r = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        r.append(e0.elapsed_time(e1) * 1e3 / n)
    return sorted(r)[2]


tot = {"quant": 0.0, "gemm": 0.0, "linear": 0.0, "bound": 0.0}
for site, K, N in synth.LLAMA3_8B_SITES:
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    q0 = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    wb = q0.codes.numel() + q0.sf.numel()
    R = max(2, (512 << 20) // wb + 1)
    qws = [q0] + [A.QWeight(N=q0.N, K=q0.K, Kp=q0.Kp, S=q0.S, layout=q0.layout, codes=q0.codes.clone(),
                            sf=q0.sf.clone(), gs=q0.gs) for _ in range(R - 1)]
    x = synth.activation(M, K, st, seed=2, device="cuda")
    c, sf = A.quantize_activation(x, prof)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ws, wsl = A.Workspace("cuda"), A.Workspace("cuda")
    tq = t(lambda i: A.quantize_activation(x, prof, c, sf), 20)
    tg = t(lambda i: A.gemm(c, sf, prof.gs, qws[i % R], out=y, ws=ws), R)
    tl = t(lambda i: A.linear(x, prof, qws[i % R], out=y, ws=wsl), R)
    bound = wb / (HBM * 1e3)
    for k, v in (("quant", tq), ("gemm", tg), ("linear", tl), ("bound", bound)):
        tot[k] += v
    print(f"[{tag}] M={M} {site:8s} quant {tq:6.2f}  gemm {tg:6.2f}  linear {tl:6.2f} us  | weights {wb / 1e6:5.1f} MB "
          f"-> {bound:5.2f} us at HBM ({R} copies)", flush=True)
    del qws, q0
    torch.cuda.empty_cache()
print(f"[{tag}] M={M} total quant {tot['quant']:.1f}  gemm {tot['gemm']:.1f}  linear {tot['linear']:.1f} us  "
      f"bound {tot['bound']:.1f} us  -> linear at {tot['bound'] / tot['linear']:.3f} of HBM")
