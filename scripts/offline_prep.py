"""the offline path at model scale (Table 4): per-site calibration statistics over
128 x 2048 tokens and ARC weight preparation for every linear layer of LLaMA-3.1-8B, Qwen2.5-7B and
Qwen2.5-32B shapes (synthetic activations / random weights -- only timing is meaningful).

Per site and layer, timed:
  calib    arc_calib_absmax over 262144 calibration rows (16 launches over a resident 16384-row chunk, the
           same bytes as the full set) + arc_select_outliers + arc_gather_order (host)
  quant    arc_tensor_scale(W) + arc_quantize_weight (reorder, NVFP4, duplicated outlier blocks)
The paper's "Calib." (79.8 s for Llama 3.1-8B on an RTX PRO 6000) also runs the FP16 model forward to
produce the activations; only its "Quant." (9.15 s) is the same work as ours.  Mem. = bytes of the
prepared linear weights (codes + block scales).  JSON on stdout."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

MODELS = {
    # name: (layers, hidden, intermediate, q_heads, kv_heads, head_dim, paper Table 4 (calib s, quant s, mem GB))
    "llama-3.1-8b": (32, 4096, 14336, 32, 8, 128, (79.84, 9.15, 4.75)),
    "qwen2.5-7b": (28, 3584, 18944, 28, 4, 128, (89.66, 9.38, 4.24)),
    "qwen2.5-32b": (64, 5120, 27648, 40, 8, 128, (176.44, 43.89, 19.57)),
}
CAL_ROWS, CHUNK = 128 * 2048, 16384
names = sys.argv[1:] or list(MODELS)


def sites(h, inter, qh, kvh, hd):
    return [("qkv", h, (qh + 2 * kvh) * hd), ("o", qh * hd, h), ("gate_up", h, 2 * inter), ("down", inter, h)]


out = {}
for name in names:
    L, h, inter, qh, kvh, hd, paper = MODELS[name]
    res = {"layers": L, "sites": {}, "paper_table4": {"calib_s": paper[0], "quant_s": paper[1], "mem_gb": paper[2]}}
    tot_cal = tot_q = 0.0
    mem = 0
    for site, K, N in sites(h, inter, qh, kvh, hd):
        st = synth.Structure(K, 128, seed=K)
        chunk = synth.activation(CHUNK, K, st, seed=1, device="cuda")
        w = synth.weight(N, K, seed=2, device="cuda")
        # warm-up (kernel attributes, allocator)
        prof = A.calibrate([chunk[:1024]])
        A.quantize_weight(w, prof)
        torch.cuda.synchronize()
        t_cal, t_q = [], []
        for layer in range(2):  # two measured layers; the rest is the same work on other data
            t0 = time.perf_counter()
            cm = None
            for _ in range(CAL_ROWS // CHUNK):
                cm = A.calib_absmax(chunk, cm)
            torch.cuda.synchronize()
            sel = A.select_outliers(cm.cpu().numpy())
            perm = A.gather_order(sel["perm"])
            prof = A.Profile(K=K, S=sel["S"], perm=torch.from_numpy(perm).cuda(),
                             gs=torch.tensor([sel["gs"]], dtype=torch.float32, device="cuda"), layout=A.INTERLEAVED)
            t1 = time.perf_counter()
            qw = A.quantize_weight(w, prof)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            t_cal.append(t1 - t0)
            t_q.append(t2 - t1)
        b = qw.codes.numel() + qw.sf.numel()
        res["sites"][site] = {"K": K, "N": N, "S": prof.S, "calib_ms_per_layer": 1e3 * min(t_cal),
                              "quant_ms_per_layer": 1e3 * min(t_q), "weight_bytes": b}
        tot_cal += min(t_cal) * L
        tot_q += min(t_q) * L
        mem += b * L
        del chunk, w, qw
        torch.cuda.empty_cache()
    res["calib_s_model"] = tot_cal
    res["quant_s_model"] = tot_q
    res["linear_weight_gb"] = mem / 1e9
    res["note"] = "per-layer minimum of 2 measured layers x layers; calib = statistics pass only (no model forward)"
    out[name] = res
    print(name, json.dumps({k: v for k, v in res.items() if k != "sites"}), file=sys.stderr)
print(json.dumps(out))
