"""Decode-size GEMM alone (arc_gemm on pre-quantized activations, weights L2-resident or HBM-cold):
per-CTA phase durations from the ARC_TRACE stamps and the SM clock implied by clock64 / globaltimer.

    ARC_TRACE=1 python scripts/trace_gemm_decode.py [M] [site]
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
want = sys.argv[2] if len(sys.argv) > 2 else "o"
name, K, N = [s for s in synth.LLAMA3_8B_SITES if s[0] == want][0]
st = synth.Structure(K, 128, seed=0)
prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
x = synth.activation(M, K, st, seed=2, device="cuda")
c, sf = A.quantize_activation(x, prof)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
ws = A.Workspace("cuda")
buf = np.zeros((64, 1024, 8), np.uint64)
for label, flush in (("L2-warm", False), ("HBM-cold", True)):
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        if flush:
            fl.zero_()
        A.gemm(c, sf, prof.gs, qw, out=y, ws=ws)
    torch.cuda.synchronize()
    lib.arc_debug_trace(buf.ctypes.data)
    if flush:
        fl.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    A.gemm(c, sf, prof.gs, qw, out=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    n = lib.arc_debug_trace(buf.ctypes.data)
    b = buf[0]
    live = b[:, 0] > 0
    t = b[live].astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t[:, :3] - t0) / 1e3
    names = ["entry", "wait", "acc"]
    med = np.median(rel, axis=0)
    mx = np.max(rel, axis=0)
    cyc = t[:, 3:7]
    cn = ["sent", "arrived", "recv", "exit"]
    print(f"M={M} {name} {label}: {int(live.sum())} CTAs; us: "
          + "  ".join(f"{nm} {m:.2f}/{x_:.2f}" for nm, m, x_ in zip(names, med, mx))
          + " | cycles after acc: " + "  ".join(f"{nm} {np.median(cyc[:, i][cyc[:, i] > 0]) if (cyc[:, i] > 0).any() else 0:.0f}"
                                                for i, nm in enumerate(cn)))
