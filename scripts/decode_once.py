"""One decode-size ARC linear per LLaMA-3-8B site (for ncu captures): python scripts/decode_once.py [M] [site]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
only = sys.argv[2] if len(sys.argv) > 2 else None
for site, K, N in synth.LLAMA3_8B_SITES:
    if only and site != only:
        continue
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=2, device="cuda")
    for _ in range(3):
        y = A.linear(x, prof, qw)
    torch.cuda.synchronize()
    print(site, float(y.float().abs().sum()))
