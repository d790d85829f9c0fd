"""Per-CTA phase stamps of the decode-size stream-K GEMM (env ARC_STREAM_TRACE=1): one arc_linear per
LLaMA-3-8B site at M tokens, HBM-cold weights; prints quantiles (us from the earliest CTA entry)."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("ARC_STREAM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

lib = A.lib()
lib.arc_debug_stream_trace.restype = ctypes.c_int
lib.arc_debug_stream_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
names = ["entry", "w-issued", "pdl-wait", "1st-stage", "last-acc", "epi-done"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for site, K, N in synth.LLAMA3_8B_SITES:
    st = synth.Structure(K, 128, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=128)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=2, device="cuda")
    ws = A.Workspace("cuda")
    for _ in range(3):
        flush.zero_()
        y = A.linear(x, prof, qw, ws=ws, mode="fused")
    torch.cuda.synchronize()
    buf = np.zeros((4096, 8), np.uint64)
    n = lib.arc_debug_stream_trace(buf.ctypes.data, 4096)
    g = int(np.count_nonzero(buf[:, 0]))
    t = buf[:g, :6].astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    rel[t == 0] = np.nan
    q = np.nanpercentile(rel, [0, 50, 100], axis=0)
    red = buf[:g, 6].astype(np.float64) / 1965.0   # cycles -> us at max clock
    pub = buf[:g, 7].astype(np.float64) / 1965.0
    print(f"M={M} {site:8s} grid {g}: " + "  ".join(f"{nm} {q[0, i]:.1f}/{q[1, i]:.1f}/{q[2, i]:.1f}"
                                                   for i, nm in enumerate(names))
          + f"  | publish(write+fence+atomic) us/CTA med {np.median(pub):.2f} max {pub.max():.2f}"
          + f"  reduce us/CTA med {np.median(red):.2f} max {red.max():.2f}", flush=True)
