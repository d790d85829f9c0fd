"""the offline path at model scale (Table 4): per-site calibration statistics over
128 x 2048 tokens and ARC weight preparation for every linear layer of LLaMA-3.1-8B, Qwen2.5-7B and
Qwen2.5-32B shapes (synthetic activations / random weights -- only timing is meaningful).  Every layer of every model is
prepared and timed (no extrapolation from a sample of layers).

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
    site_list = sites(h, inter, qh, kvh, hd)
    chunks = {}
    for site, K, N in site_list:  # one resident calibration chunk per distinct K (synthetic activations)
        if K not in chunks:
            chunks[K] = synth.activation(CHUNK, K, synth.Structure(K, 128, seed=K), seed=1, device="cuda")
    for site, K, N in site_list:  # warm-up (kernel attributes, allocator)
        prof = A.calibrate([chunks[K][:1024]])
        A.quantize_weight(synth.weight(N, K, seed=2, device="cuda"), prof)
    torch.cuda.synchronize()
    t_cal = {s: [] for s, _, _ in site_list}
    t_q = {s: [] for s, _, _ in site_list}
    prepared = []  # every layer's prepared weights stay resident: Mem. is what the model actually holds
    for layer in range(L):
        for site, K, N in site_list:
            w = synth.weight(N, K, seed=1000 * layer + K + N, device="cuda")  # untimed: the checkpoint load
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cm = None
            for _ in range(CAL_ROWS // CHUNK):
                cm = A.calib_absmax(chunks[K], cm)
            torch.cuda.synchronize()
            sel = A.select_outliers(cm.cpu().numpy())
            perm = A.gather_order(sel["perm"])
            prof = A.Profile(K=K, S=sel["S"], perm=torch.from_numpy(perm).cuda(),
                             gs=torch.tensor([sel["gs"]], dtype=torch.float32, device="cuda"), layout=A.INTERLEAVED)
            t1 = time.perf_counter()
            qw = A.quantize_weight(w, prof)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            t_cal[site].append(t1 - t0)
            t_q[site].append(t2 - t1)
            prepared.append(qw)
            del w
            if layer == 0:
                res["sites"][site] = {"K": K, "N": N, "S": prof.S, "weight_bytes": qw.codes.numel() + qw.sf.numel()}
    for site, _, _ in site_list:
        res["sites"][site]["calib_ms_per_layer_median"] = 1e3 * float(np.median(t_cal[site]))
        res["sites"][site]["quant_ms_per_layer_median"] = 1e3 * float(np.median(t_q[site]))
    res["calib_s_model"] = float(sum(sum(v) for v in t_cal.values()))
    res["quant_s_model"] = float(sum(sum(v) for v in t_q.values()))
    res["linear_weight_gb"] = sum(q.codes.numel() + q.sf.numel() for q in prepared) / 1e9
    res["note"] = ("every layer measured (sum of per-layer wall times, no extrapolation); calib = statistics pass over "
                   "128 x 2048 rows per site and layer + outlier selection + gather order, no model forward; "
                   "quant = tensor scale + reorder + NVFP4 + duplicated outlier blocks; all prepared weights resident")
    out[name] = res
    print(name, json.dumps({k: v for k, v in res.items() if k != "sites"}), file=sys.stderr)
    del prepared, chunks
    torch.cuda.empty_cache()
print(json.dumps(out))
