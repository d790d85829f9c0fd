"""Per-CTA finish times of the prefill GEMM (ARC_TRACE=1) split by the size of the cluster the CTA ran in
(preferred clusters of 4 vs fallback pairs): shows whether a static tile schedule leaves the faster
4-CTA clusters idle while the pairs finish."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("ARC_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

lib = A.lib()
lib.arc_debug_trace.restype = ctypes.c_int
lib.arc_debug_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros((64, 1024, 8), np.uint64)
for name, K, N in synth.LLAMA3_8B_SITES:
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(8192, K, st, seed=2, device="cuda")
    c, sf = A.quantize_activation(x, prof)
    y = torch.empty(8192, N, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        A.gemm(c, sf, prof.gs, qw, out=y)
    torch.cuda.synchronize()
    lib.arc_debug_trace(buf.ctypes.data)
    A.gemm(c, sf, prof.gs, qw, out=y)
    torch.cuda.synchronize()
    n = lib.arc_debug_trace(buf.ctypes.data)
    b = buf[n - 1]
    live = b[:, 1] > 0
    t0 = b[live, 0].min()
    ex = (b[live, 1].astype(np.float64) - t0) / 1e3
    nct = b[live, 2]
    out = []
    for k in sorted(set(nct.tolist())):
        e = ex[nct == k]
        out.append(f"cluster {k}: {e.size} CTAs exit min/med/max {e.min():.1f}/{np.median(e):.1f}/{e.max():.1f} us")
    print(f"{name}: " + " | ".join(out), flush=True)
