import os, sys, torch, numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from paper_2601_07475_b200 import arc as A, synth
for (M, N, K) in [(1, 4096, 4096), (16, 4096, 4096), (16, 6144, 4096), (16, 512, 4096), (16, 384, 1024), (4, 1024, 4096), (16, 1024, 1024), (16, 512, 2048)]:
    st = synth.Structure(K, 128, seed=1)
    x = synth.activation(M, K, st, seed=2, device="cuda")
    w = synth.weight(N, K, seed=3, device="cuda")
    prof = A.calibrate([synth.activation(256, K, st, seed=4, device="cuda")], s_override=128)
    qw = A.quantize_weight(w, prof)
    codes, sf = A.quantize_activation(x, prof)
    y1 = A.gemm(codes, sf, prof.gs, qw, out_dtype=torch.float32, ws=A.Workspace("cuda"))
    torch.cuda.synchronize()
    yref, bound = oracle.gemm_reference(codes.cpu().numpy(), sf.cpu().numpy(), qw.codes.cpu().numpy(), qw.sf.cpu().numpy(), float(prof.gs.item()), float(qw.gs.item()))
    r = np.abs(y1.cpu().numpy() - yref) / np.maximum(bound, 1e-30)
    per_tile = r.reshape(M, -1, 128).max(axis=(0, 2)) if N % 128 == 0 else r.max(axis=0)
    per_row = r.max(axis=1)
    nkb = (K + 128 + 255) // 256
    print(f"M={M} N={N} K={K} nkb={nkb}: worst {r.max():.3g}; bad tiles {np.nonzero(per_tile > 1)[0].tolist()[:24]}; bad rows {np.nonzero(per_row > 1)[0].tolist()}", flush=True)
