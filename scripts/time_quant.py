"""Time arc_quantize_activation alone (CUDA events, L2-cold inputs by rotation)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--S", type=int, default=128)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--norm", action="store_true", help="time arc_rmsnorm_quantize_activation (fused RMSNorm)")
ap.add_argument("--silu", action="store_true", help="time arc_silu_mul_quantize_activation (fused SiLU-mul)")
ap.add_argument("--pairs", action="store_true", help="with --silu: gate/up as adjacent pairs (ARC_GU_PAIRS)")
ap.add_argument("--mx", action="store_true", help="time arc_quantize_activation_mx (MXFP4-ARC)")
args = ap.parse_args()
K, M, S = args.K, args.M, args.S
st = synth.Structure(K, S, seed=0)
prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=S,
                  gather_bytes=4 if args.pairs else 2)
nrot = max(2, int(4 * 126e6 // (M * K * 2)) + 1)
if args.silu:
    nrot = max(2, int(4 * 126e6 // (M * K * 4)) + 1)
    xs = [synth.gate_up(M, K, st, seed=i, device="cuda") for i in range(nrot)]
    if args.pairs:  # (g_j, u_j) adjacent
        xs = [torch.stack([x[:, :K], x[:, K:]], dim=2).reshape(M, 2 * K).contiguous() for x in xs]
else:
    xs = [synth.activation(M, K, st, seed=i, device="cuda") for i in range(nrot)]
gamma = synth.rmsnorm_weight(K, seed=0, device="cuda")
if args.norm:
    def quant(x, prof, codes=None, sf=None):
        return A.rmsnorm_quantize_activation(x, gamma, 1e-5, prof, codes, sf)
elif args.mx:
    prof = A.mx_profile(prof, float(xs[0].float().abs().max()))
    quant = A.quantize_activation_mx
elif args.silu:
    def quant(x, prof, codes=None, sf=None):
        return A.silu_mul_quantize_activation(x, prof, up_off=A.GU_PAIRS if args.pairs else None, codes=codes, sf=sf)
else:
    quant = A.quantize_activation
codes, sf = quant(xs[0], prof)
for i in range(3):
    quant(xs[i % nrot], prof, codes, sf)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    quant(xs[0], prof, codes, sf)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(nrot):
            quant(xs[i], prof, codes, sf)
torch.cuda.synchronize()
ts = []
for it in range(max(3, args.iters // nrot)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / nrot)
ts.sort()
Kp = codes.shape[1] * 2
byts = M * ((4 if args.silu else 2) * K + Kp // 2 + Kp // 16)
med = ts[len(ts) // 2]
print(f"{'rmsnorm+quant' if args.norm else 'silu+quant' if args.silu else 'mx-quant' if args.mx else 'quant'} K={K} M={M} S={S}: median {med*1e3:.1f} us  {byts/med/1e6:.0f} GB/s  (min {ts[0]*1e3:.1f} us)")

# reference: plain torch streaming kernels on the same rotated buffers
def _t(fn):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.iters)]
    for i in range(args.iters):
        e[2 * i].record()
        fn(i)
        e[2 * i + 1].record()
    torch.cuda.synchronize()
    return sorted(e[2 * i].elapsed_time(e[2 * i + 1]) for i in range(args.iters))[args.iters // 2]


dst = torch.empty_like(xs[0])
t = _t(lambda i: dst.copy_(xs[i % nrot]))
print(f"torch copy_ of x ({M*K*2/1e6:.0f} MB read + write): {t*1e3:.1f} us  {2*M*K*2/t/1e6:.0f} GB/s")
acc = torch.empty(M, dtype=torch.float32, device="cuda")
t = _t(lambda i: torch.amax(xs[i % nrot], dim=1, out=acc.to(torch.bfloat16)) if False else xs[i % nrot].view(torch.int32).sum(dim=1))
print(f"torch int32 row-sum of x (read only): {t*1e3:.1f} us  {M*K*2/t/1e6:.0f} GB/s")
