"""Context only: cuBLASLt NVFP4 GEMM (torch._scaled_mm) on the same packed operands/shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_07475_b200 import arc as A, synth  # noqa: E402

for site, K, N in synth.LLAMA3_8B_SITES:
    M, S = 8192, 128
    st = synth.Structure(K, S, seed=0)
    prof = A.calibrate([synth.activation(1024, K, st, seed=1000, device="cuda")], s_override=S)
    qw = A.quantize_weight(synth.weight(N, K, seed=1, device="cuda"), prof)
    x = synth.activation(M, K, st, seed=2, device="cuda")
    codes, sf = A.quantize_activation(x, prof)
    a = codes.view(torch.float4_e2m1fn_x2)
    b = qw.codes.view(torch.float4_e2m1fn_x2)
    f = lambda: torch._scaled_mm(a, b.t(), scale_a=sf.view(torch.float8_e4m3fn),
                                 scale_b=qw.sf.view(torch.float8_e4m3fn), out_dtype=torch.bfloat16)
    try:
        for _ in range(3):
            f()
    except Exception as e:
        print(site, "unavailable:", str(e)[:200])
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    fl = 2.0 * M * N * (K + S)
    print(f"cublasLt nvfp4 {site}: {t*1e3:.1f} us {fl/t/1e9:.0f} TFLOP/s")
    bf = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    wb = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    g = lambda: bf @ wb.t()
    for _ in range(3):
        g()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"cublas bf16 {site}: {t*1e3:.1f} us {2.0*M*N*K/t/1e9:.0f} TFLOP/s")
