"""Decode-size (M=16) per-kernel latency of one ARC linear site in CUDA graphs: quantize alone,
GEMM (+ split-K reduce) alone, and the full arc_linear chain, 20 calls per replay."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16


def t(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
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


for site, K, N in synth.LLAMA3_8B_SITES:
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=2, device="cuda")
    c, sf = A.quantize_activation(x, prof)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ws = A.Workspace("cuda")
    wsl = A.Workspace("cuda")
    tq = t(lambda: A.quantize_activation(x, prof, c, sf))
    tg = t(lambda: A.gemm(c, sf, prof.gs, qw, out=y, ws=ws))
    tl = t(lambda: A.linear(x, prof, qw, out=y, ws=wsl))
    print(f"M={M} {site:8s} quant {tq:6.2f} us  gemm(+reduce) {tg:6.2f} us  linear {tl:6.2f} us  "
          f"(weights {qw.codes.numel() / 1e6:.1f} MB, L2-warm)")
