"""Timeline of the decode-size 4-site step (env ARC_TRACE=1): every quantize and decode-GEMM launch
records per-CTA globaltimer stamps; one CUDA-graph replay of the step (weights HBM-cold, as in the
bench) is traced and each launch is summarised relative to the step's first stamp (us):
first entry / median entry, griddepcontrol.wait passed (min/median/max), acc ready (GEMM), last exit.

    ARC_TRACE=1 [MODEL=70b] python scripts/trace_decode.py [M]
"""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("ARC_TRACE", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

lib = A.lib()
lib.arc_debug_trace.restype = ctypes.c_int
lib.arc_debug_trace.argtypes = [ctypes.c_void_p]
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mode = os.environ.get("MODE", "unfused")
SITES = synth.LLAMA3_70B_SITES if os.environ.get("MODEL", "8b") == "70b" else synth.LLAMA3_8B_SITES

sites = []
for name, K, N in SITES:
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    sites.append((name, K, N, prof, qw))
xs = [synth.activation(M, K, synth.Structure(K, 8, seed=5), seed=9, device="cuda") for _, K, *_ in sites]
ys = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _, _, N, *_ in sites]
wss = [A.Workspace("cuda") for _ in sites]


def step():
    for (name, K, N, prof, qw), x, y, ws in zip(sites, xs, ys, wss):
        A.linear(x, prof, qw, out=y, ws=ws, mode=mode)


step()
torch.cuda.synchronize()
buf = np.zeros((64, 1024, 8), np.uint64)
lib.arc_debug_trace(buf.ctypes.data)  # discard the warm-up / calibration launches
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        step()
torch.cuda.synchronize()
n = lib.arc_debug_trace(buf.ctypes.data)  # the launches captured into the graph (slots 0 .. n-1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
lib.arc_debug_trace(buf.ctypes.data)
print(f"M={M} mode={mode}: {n} traced launches in the graph")
t0 = min(int(buf[i][buf[i][:, 0] > 0][:, 0].min()) for i in range(n) if (buf[i][:, 0] > 0).any())
for i in range(n):
    b = buf[i]
    live = b[:, 0] > 0
    if not live.any():
        print(f"  launch {i}: no stamps")
        continue
    t = (b[live].astype(np.float64) - t0) / 1e3
    t[b[live] == 0] = np.nan
    kind = "quant" if i % 2 == 0 else "gemm "
    site = sites[i // 2][0]

    def q(c):
        v = t[:, c]
        v = v[~np.isnan(v)]
        return (f"{v.min():6.2f}/{np.median(v):6.2f}/{v.max():6.2f}" if v.size else "   -   ")
    if kind == "quant":
        names = ["entry", "wait", "prod-done", "prim-done"]
        print(f"  {site:8s} {kind} ctas {int(live.sum()):4d}  " + "  ".join(f"{nm} {q(c)}" for c, nm in enumerate(names)))
    else:
        cyc = b[live][:, 3:7].astype(np.float64)
        cn = ["sent", "bulk", "recv", "done"]
        print(f"  {site:8s} {kind} ctas {int(live.sum()):4d}  " + "  ".join(f"{nm} {q(c)}" for c, nm in enumerate(["entry", "wait", "acc"]))
              + " | cyc after acc (med/max): " + "  ".join(
                  f"{nm} {np.median(cyc[:, i][cyc[:, i] > 0]):.0f}/{cyc[:, i].max():.0f}" if (cyc[:, i] > 0).any() else f"{nm} -"
                  for i, nm in enumerate(cn)))
