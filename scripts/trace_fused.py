"""Per-CTA timeline of the fused decode linear (timing experiments only): run with
ARC_FUSED_TRACE=1; each site is replayed in a CUDA graph over rotating weight copies (as in
time_decode.py) and the globaltimer stamps of the last launch are summarised (us, relative
to the first CTA's entry): 0 entry, 1 prologue done, 2 griddepcontrol.wait passed, 3 phase-1
quantize done, 4 grid barrier passed (producer), 5 first stage full (MMA), 6 last MMA issued,
7 exit."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

lib = A.lib()
lib.arc_debug_fused_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
S = 128
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
for site, K, N in synth.LLAMA3_8B_SITES:
    st = synth.Structure(K, S, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=S)
    w = synth.weight(N, K, seed=1, device="cuda")
    qws = [A.quantize_weight(w, prof) for _ in range(max(2, int(4 * 126e6 // (N * K * 0.6)) + 1))]
    x = synth.activation(M, K, st, seed=2, device="cuda")
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ws = A.Workspace("cuda")
    for q in qws[:2]:
        A.linear(x, prof, q, out=y, ws=ws, mode="fused")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for q in qws:
                A.linear(x, prof, q, out=y, ws=ws, mode="fused")
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    buf = np.zeros((4096, 8), np.uint64)
    n = lib.arc_debug_fused_trace(buf.ctypes.data, 4096)
    tr = buf[:148].astype(np.int64)
    tr = tr[tr[:, 0] > 0]
    t = (tr - tr[:, 0].min()) / 1e3
    names = ["entry", "prolog", "pdlwait", "quant", "barrier", "full0", "lastmma", "exit"]
    print(f"{site} M={M} N={N} K={K} ctas={len(tr)} (us from first entry; min / median / max)")
    for i, nm in enumerate(names):
        print(f"   {nm:8s} {t[:, i].min():7.2f} {np.median(t[:, i]):7.2f} {t[:, i].max():7.2f}")
    del qws
