"""Fig.8a analogue (caption P:394-396): GEMM latency vs the augmented channel count S for
ARC-NVFP4 (K+S, the hot path), native MXFP4-ARC (K+S, tcgen05 kind::mxf4), and the S-independent comparison
GEMMs W4A8 (MXFP8 activations x MXFP4 weights) and MXFP8 (both on kind::mxf8f6f4) -> JSON on stdout.

Every GEMM is timed alone in a CUDA graph of `reps` launches (median of 5 replays); inputs are synthetic
(synth.py recipe) at the LLaMA-3-8B and Qwen2.5-7B linear shapes; bf16 output."""
import argparse
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
    del g
    return sorted(ts)[2] * 1e3  # us


ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, nargs="+", default=[2048, 8192])
ap.add_argument("--S", type=int, nargs="+", default=[0, 64, 128, 256, 512, 1024, 2048])
ap.add_argument("--models", nargs="+", default=["llama-3-8b", "qwen2.5-7b"])
args = ap.parse_args()
SHAPES = {"llama-3-8b": list(synth.LLAMA3_8B_SITES),
          "qwen2.5-7b": [("qkv", 3584, 4608), ("o", 3584, 3584), ("gate_up", 3584, 37888), ("down", 18944, 3584)]}
out = {"what": "Fig.8a analogue: GEMM latency (us) vs S; comparators are S-independent", "runs": []}
ws = A.Workspace("cuda")
for model in args.models:
    for site, K, N in SHAPES[model]:
        w = synth.weight(N, K, seed=1, device="cuda")
        for M in args.M:
            st = synth.Structure(K, 128, seed=0)
            x = synth.activation(M, K, st, seed=2, device="cuda")
            y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            rec = {"model": model, "site": site, "M": M, "K": K, "N": N, "arc_nvfp4": [], "arc_mx_native": []}
            # comparators (K only)
            a8, a8sf = A.quantize_mxfp8(x)
            b8, b8sf = A.quantize_mxfp8(w)
            rec["mxfp8_us"] = graph_time(lambda: A.gemm_mxfp8(a8, a8sf, b8, b8sf, K, out=y, ws=ws))
            ident = A.profile_from(np.arange(K, dtype=np.int32), 0, 1.0)
            b4, b4sf = A.quantize_mx_native(w, ident, weight=True)
            rec["w4a8_us"] = graph_time(lambda: A.gemm_w4a8(a8, a8sf, b4, b4sf, K, out=y, ws=ws))
            del b8, b8sf, b4, b4sf
            base = A.calibrate([x[:1024]], s_override=0)  # one channel order; S only moves the boundary
            perm = base.perm.cpu().numpy()
            for S in args.S:
                if S > K:
                    continue
                prof = A.profile_from(perm, S, float(base.gs.item()))
                qw = A.quantize_weight(w, prof)
                codes, sf = A.quantize_activation(x, prof)
                t = graph_time(lambda: A.gemm(codes, sf, prof.gs, qw, out=y, ws=ws))
                rec["arc_nvfp4"].append({"S": S, "us": t, "tflops_KS": 2.0 * M * N * (K + S) / t / 1e6})
                del qw, codes, sf
                mc, msf = A.quantize_mx_native(x, prof)
                mw, mwsf = A.quantize_mx_native(w, prof, weight=True)
                t = graph_time(lambda: A.gemm_mx_native(mc, msf, mw, mwsf, out=y, ws=ws))
                rec["arc_mx_native"].append({"S": S, "us": t})
                del mc, msf, mw, mwsf
                torch.cuda.empty_cache()
            for key in ("arc_nvfp4", "arc_mx_native"):
                Ss = np.array([r["S"] for r in rec[key]], float)
                ts = np.array([r["us"] for r in rec[key]])
                slope, icpt = np.polyfit(Ss, ts, 1)
                pred = slope * Ss + icpt
                rec[key + "_fit"] = {"us_per_channel": slope, "us_at_S0": icpt,
                                     "r2": float(1 - np.sum((ts - pred) ** 2) / np.sum((ts - ts.mean()) ** 2))}
            s128 = next((r["us"] for r in rec["arc_nvfp4"] if r["S"] == 128), None)
            rec["arc_s128_vs_w4a8"] = rec["w4a8_us"] / s128 if s128 else None
            rec["arc_s128_vs_mxfp8"] = rec["mxfp8_us"] / s128 if s128 else None
            out["runs"].append(rec)
            print(model, site, M, "nvfp4", [round(r["us"], 1) for r in rec["arc_nvfp4"]], "mx",
                  [round(r["us"], 1) for r in rec["arc_mx_native"]], "w4a8 %.1f mxfp8 %.1f" %
                  (rec["w4a8_us"], rec["mxfp8_us"]), file=sys.stderr, flush=True)
            del x, y, a8, a8sf
            torch.cuda.empty_cache()
        del w
print(json.dumps(out))
