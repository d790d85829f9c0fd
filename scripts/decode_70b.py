"""LLaMA-3-70B layer decode sweep (BASELINE configs[3] shapes on one GPU, 488 MB of weights per 4-site step)
through bench.py's own decode_sweep, at M = 1 / 16 / 32 / 64; ARC_* environment variables select kernel
variants for A/B runs.

    python scripts/decode_70b.py
"""
import json, os, sys
sys.argv = ["x"]
sys.path.insert(0, ".")
import torch
import bench
from paper_2601_07475_b200 import arc as A
dev = torch.device("cuda", 0)
peaks = bench._peaks()
s70 = bench.build_sites(A, 128, 0, 1, dev, workload="llama3-70b", cal_rows=1024)
r = bench.decode_sweep(A, s70, dev, peaks, Ms=(1, 16, 32, 64))
print("WAVE1=" + os.environ.get("ARC_DECODE_WAVE1", "1"),
      json.dumps([(x["M_tokens"], round(x["us_per_layer_step"], 1), round(x["hbm_frac"], 3)) for x in r]))
