"""Decode-size LLaMA-3-8B layer step (4 ARC linears) with and without cross-linear L2 weight prefetch
(arc_prefetch_l2 one linear ahead).  Each graph replay walks R copies of the layer's weights (R x 128 MB
>= 3x L2), so every step streams its weights from HBM.  Prints us per layer step and the HBM fraction."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
R = 3
Ms = [int(a) for a in sys.argv[1:]] or [1, 4, 16, 32, 64]
sites = []
for name, K, N in synth.LLAMA3_8B_SITES:
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    q0 = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    qws = [q0] + [A.QWeight(N=q0.N, K=q0.K, Kp=q0.Kp, S=q0.S, layout=q0.layout, codes=q0.codes.clone(),
                            sf=q0.sf.clone(), gs=q0.gs) for _ in range(R - 1)]
    sites.append((name, K, N, prof, qws))
wbytes = sum(q[0].codes.numel() + q[0].sf.numel() for *_, q in sites)


def run(M, mode, pf):
    xs = [synth.activation(M, K, synth.Structure(K, 8, seed=5), seed=9, device="cuda") for _, K, *_ in sites]
    ys = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _, _, N, *_ in sites]
    wss = [A.Workspace("cuda") for _ in sites]

    def step(r):
        if pf == "all":
            for *_, qws in sites:
                A.prefetch_weights(qws[r])
        for i, ((_, _, _, prof, qws), x, y, ws) in enumerate(zip(sites, xs, ys, wss)):
            if pf == "next":
                if i == 0:
                    A.prefetch_weights(qws[r])
                if i + 1 < len(sites):
                    A.prefetch_weights(sites[i + 1][4][r])
            A.linear(x, prof, qws[r], out=y, ws=ws, mode=mode)

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for r in range(R):
            step(r)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for r in range(R):
                step(r)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    us = sorted(ts)[3]
    db = wbytes + sum(M * K * 2 + M * N * 2 for _, K, N, *_ in sites)
    return us, db / (us * 1e-6) / 1e9 / HBM


res = []
for M in Ms:
    for mode in ("auto", "unfused", "fused"):
        for pf in ("none", "next", "all"):
            us, frac = run(M, mode, pf)
            res.append({"M": M, "mode": mode, "prefetch": pf, "us": us, "hbm_frac": frac})
            print(f"M={M:3d} {mode:8s} prefetch={pf:5s} {us:7.1f} us  {frac:.3f} of HBM", flush=True)
print(json.dumps({"weight_bytes": wbytes, "hbm_gbs": HBM, "runs": res}))
