#!/usr/bin/env python
"""Benchmark of the ARC-NVFP4 linear hot path on B200 (BASELINE.json metric:
"ARC NVFP4 linear TFLOPS (% FP4 tensor peak) + quantize HBM GB/s, 1/2/4/8 GPU").

One step = the four ARC linear sites of one LLaMA-3-8B decoder layer at prefill
(BASELINE.json configs[1]): fused qkv (K=4096 -> N=6144), o (4096 -> 4096), fused
gate-up (4096 -> 28672), down (14336 -> 4096), M = 8192 tokens, S = 128 augmented
channels each; every site = arc_quantize_activation + arc_gemm (what arc_linear
runs).  Synthetic activations with injected outlier channels, random weights
(DESIGN.md "Input recipe"); per-step footprint (~0.6 GB) is far above the 126 MB L2.

N > 1 (torchrun): Megatron-style tensor parallelism of the same layer (strong
scaling): qkv / gate-up column-parallel over N (no communication), o / down
row-parallel over K with per-rank calibration and an NCCL all-reduce of Y.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl arc|reference] [--M 8192]
"""
from __future__ import annotations

import argparse
import json
import zlib
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2601_07475_b200 import synth  # noqa: E402

SITES = synth.LLAMA3_8B_SITES
S_AUG = 128


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- workload
class Site:
    def __init__(self, name, K, N, M, S, rank, world, mode, device, A, layout="mp"):
        """mode: 'full' (1 GPU), 'col' (column-parallel shard of N), 'row' (row-parallel shard of K).
        Sharded sites are built with paper_2601_07475_b200.tp (the tested host logic).  layout 'sp'
        (sequence parallel): a col site quantizes its M/P token rows and all-gathers the
        packed codes + scales; a row site reduce-scatters its output over tokens.  'mp': a col site
        quantizes the replicated M rows; a row site all-reduces."""
        from paper_2601_07475_b200 import tp
        self.name, self.M, self.mode = name, M, mode
        self.sp = layout == "sp" and world > 1
        seed = zlib.crc32(name.encode()) % 1000
        st = synth.Structure(K, S, seed=seed * 31)
        cal = synth.activation(4096, K, st, seed=seed + 1000, device=device)
        w = synth.weight(N, K, seed=seed * 7, device=device)
        x = synth.activation(M, K, st, seed=seed + 1, device=device)
        if mode == "full":
            self.prof = A.calibrate([cal], s_override=S)
            self.qw = A.quantize_weight(w, self.prof)
            self.x = x
        elif mode == "col":
            prof = A.calibrate([cal], s_override=S)
            lin = tp.ColumnParallelLinear(w, prof, rank, world, backend=A)
            self.prof, self.qw, self.x = lin.profile, lin.qweight, x
        else:
            S_r = max(16, (S // world + 15) // 16 * 16)
            lin = tp.RowParallelLinear(w, cal, rank, world, s_override=S_r, backend=A)
            self.prof, self.qw = lin.profile, lin.qweight
            self.x = x[:, lin.shard.lo:lin.shard.hi].contiguous()
        del cal, w, x
        Kl, Nl, S_l = self.prof.K, self.qw.N, self.prof.S
        self.K, self.N, self.S = Kl, Nl, S_l
        self.gs_w = float(self.qw.gs.item())
        Kp, cb, sb = A.buffer_sizes(M, Kl, S_l)
        self.Kp = Kp
        self.codes = torch.empty(M, Kp // 2, dtype=torch.uint8, device=device)
        self.sf = torch.empty(sb, dtype=torch.uint8, device=device)
        self.y = torch.empty(M, Nl, dtype=torch.bfloat16, device=device)
        self.m_q = M  # rows this rank quantizes
        if self.sp and mode == "col":
            ml = M // world
            assert ml % 128 == 0, "sequence-parallel rows per rank must be a multiple of 128"
            self.x = self.x[rank * ml:(rank + 1) * ml].contiguous()
            self.codes_loc = torch.empty(ml, Kp // 2, dtype=torch.uint8, device=device)
            self.sf_loc = torch.empty(ml * Kp // 16, dtype=torch.uint8, device=device)
            self.m_q = ml
        if self.sp and mode == "row":
            self.y_rs = torch.empty(M // world, Nl, dtype=torch.bfloat16, device=device)
        self.ws = A.Workspace(device)
        self.flops = 2.0 * M * Nl * (Kl + S_l)                       # SPEC S:322 cost model, algorithmic
        self.flops_eff = 2.0 * M * Nl * Kl
        self.q_bytes = self.m_q * (2 * Kl + Kp // 2 + Kp // 16) + 4 * Kl  # bf16 read + codes + scales + perm
        self.g_bytes = Nl * Kp * 9 // 16 + M * Kp * 9 // 16 + M * Nl * 2


def build_sites(A, M, rank, world, device, layout="mp"):
    sites = []
    for name, K, N in SITES:
        if world == 1:
            mode = "full"
        else:
            mode = "col" if name in ("qkv", "gate_up") else "row"
        sites.append(Site(name, K, N, M, S_AUG, rank, world, mode, device, A, layout))
    return sites


def run_step(A, sites, ev=None, pg=None):
    for i, s in enumerate(sites):
        if ev is not None:
            ev[i][0].record()
        if s.sp and s.mode == "col":
            # sequence parallel: quantize this rank's token rows, all-gather the packed codes + scales
            A.quantize_activation(s.x, s.prof, s.codes_loc, s.sf_loc)
            torch.distributed.all_gather_into_tensor(s.codes, s.codes_loc, group=pg)
            torch.distributed.all_gather_into_tensor(s.sf, s.sf_loc, group=pg)
        else:
            A.quantize_activation(s.x, s.prof, s.codes, s.sf)
        if ev is not None:
            ev[i][1].record()
        A.gemm(s.codes, s.sf, s.prof.gs, s.qw, out=s.y, ws=s.ws)
        if ev is not None:
            ev[i][2].record()
        if s.mode == "row" and pg is not None:
            if s.sp:
                torch.distributed.reduce_scatter_tensor(s.y_rs, s.y, group=pg)
            else:
                torch.distributed.all_reduce(s.y, group=pg)


# ----------------------------------------------------------------------------- oracle (CPU) legs
def oracle_sample(sites_meta, rows_per_site=4, budget_s=20.0):
    """Time the oracle (plain C, single thread) on a bounded sample of the same
    workload: for each site, ARC-quantize `rows_per_site` activation rows and run
    the exact GEMM of those rows against the site's full weight.  Returns
    (TFLOP/s in the bench's unit, description, seconds)."""
    import oracle
    oracle.build()
    t_total, flops_total, done = 0.0, 0.0, []
    for (name, K, N, S, xbits, perm, gs, wcodes, wsf, gs_w) in sites_meta:
        t0 = time.perf_counter()
        ac, asf = oracle.quantize_activation(xbits, perm, S, gs)
        oracle.gemm_reference(ac, asf, wcodes, wsf, gs, gs_w)
        dt = time.perf_counter() - t0
        t_total += dt
        flops_total += 2.0 * xbits.shape[0] * N * (K + S)
        done.append(f"{name}:{xbits.shape[0]}x{N}x{K}+{S}")
        if t_total > budget_s:
            break
    return flops_total / t_total / 1e12, ";".join(done), t_total


def sites_meta_for_oracle(sites, rows):
    from oracle import as_bf16_bits
    meta = []
    for s in sites:
        xb = as_bf16_bits(s.x[:rows].cpu())
        meta.append((s.name, s.K, s.N, s.S, xb, s.prof.perm.cpu().numpy(), float(s.prof.gs.item()),
                     s.qw.codes.cpu().numpy(), s.qw.sf.cpu().numpy(), s.gs_w))
    return meta


def traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="arc", choices=["arc", "reference"])
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--tp-layout", default="mp", choices=["mp", "sp"],
                    help="N>1: sequence-parallel (quantize M/P rows + all-gather packed codes, reduce-scatter) "
                         "or plain Megatron (replicated quantize, all-reduce)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = torch.distributed.group.WORLD
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    peaks = _peaks()
    fp4_peak_sus = peaks["bf16_sus"] * 4.0   # guide nominal ratio fp4/bf16 = 9/2.25
    fp4_peak_burst = peaks["bf16"] * 4.0
    workload = "llama3-8b-layer-4-arc-linears-prefill"
    config = {"workload": workload, "M_tokens": args.M, "S": S_AUG,
              "sites": [f"{n}:K{k}xN{nn}" for n, k, nn in SITES],
              "parallelism": "single" if world == 1 else f"tp{world}-{args.tp_layout}",
              "l2": "per-step footprint > 4x L2 (no flush needed)"}

    if args.impl == "reference":
        # the oracle on the host cores, same metric/config, bounded sample per step
        if rank != 0:
            return
        from paper_2601_07475_b200 import arc as A
        sites = build_sites(A, 64, 0, 1, device)
        meta = sites_meta_for_oracle(sites, 1)
        for _ in range(args.warmup if args.warmup < 1 else 0):
            pass
        vals = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            v, desc, secs = oracle_sample(meta, budget_s=30.0)
            vals.append(v)
        el = time.perf_counter() - t0
        v = float(np.median(vals))
        line = {"impl": "reference", "metric": "ARC NVFP4 linear TFLOPS", "value": v, "unit": "TFLOP/s",
                "n_gpus": 1, "steps": args.steps, "warmup": 0, "ms_per_step": el / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64-exact (oracle)",
                "data": "synthetic", "config": config,
                "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": 1, "kind": "oracle",
                                 "sample": f"1 row per site, full N: {desc}"},
                "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    from paper_2601_07475_b200 import arc as A
    if not A.device_supported():
        raise SystemExit("bench.py: current device is not sm_100 -- the ARC path has no fallback")
    sites = build_sites(A, args.M, rank, world, device, args.tp_layout)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        run_step(A, sites, pg=pg)
    torch.cuda.synchronize()

    nS = len(sites)
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(nS)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if pg is not None:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        start.record()
        for k in range(args.steps):
            run_step(A, sites, ev=evs[k], pg=pg)
        stop.record()
        torch.cuda.synchronize()
    if pg is not None:
        torch.distributed.barrier()
    ms = start.elapsed_time(stop)
    q_ms = sum(evs[k][i][0].elapsed_time(evs[k][i][1]) for k in range(args.steps) for i in range(nS)) / args.steps
    g_ms = sum(evs[k][i][1].elapsed_time(evs[k][i][2]) for k in range(args.steps) for i in range(nS)) / args.steps
    per_site = {s.name: {"gemm_us": 1e3 * sum(evs[k][i][1].elapsed_time(evs[k][i][2]) for k in range(args.steps))
                         / args.steps,
                         "quant_us": 1e3 * sum(evs[k][i][0].elapsed_time(evs[k][i][1]) for k in range(args.steps))
                         / args.steps} for i, s in enumerate(sites)}
    if pg is not None:
        t = torch.tensor([ms, q_ms, g_ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, q_ms, g_ms = t.tolist()

    flops_rank = sum(s.flops for s in sites)
    # whole-job units: TP shards one layer; each rank's flops are disjoint parts of it
    flops_job = flops_rank * world
    ms_step = ms / args.steps
    value = flops_job / (ms_step * 1e-3) / 1e12
    g_tflops = flops_rank / (g_ms * 1e-3) / 1e12
    q_bytes = sum(s.q_bytes for s in sites)
    q_gbs = q_bytes / (q_ms * 1e-3) / 1e9
    for s in sites:
        s_ = per_site[s.name]
        s_["gemm_tflops"] = s.flops / (s_["gemm_us"] * 1e-6) / 1e12
        s_["quant_gbs"] = s.q_bytes / (s_["quant_us"] * 1e-6) / 1e9

    out = {"metric": "ARC NVFP4 linear TFLOPS", "value": value, "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "nvfp4(e2m1+ue4m3)->fp32acc->bf16",
           "data": "synthetic (LLaMA-3-8B shapes, injected outlier channels, random weights)", "config": config,
           "roofline": {"bound": "tensor", "kernel": "arc_gemm_kernel (4 launches/step)",
                        "achieved": g_tflops, "peak": fp4_peak_sus, "unit": "TFLOP/s", "frac": g_tflops / fp4_peak_sus,
                        "peak_note": f"{peaks['src']} bf16 sustained {peaks['bf16_sus']} x 4 (fp4/bf16 nominal 9/2.25); "
                                     f"burst x4 = {fp4_peak_burst:.0f}, frac_burst = {g_tflops / fp4_peak_burst:.3f}",
                        "traffic": None},
           "quantize": {"bound": "hbm", "kernel": "arc_quant_kernel (4 launches/step)", "achieved": q_gbs,
                        "peak": peaks["hbm"], "unit": "GB/s", "frac": q_gbs / peaks["hbm"],
                        "bytes_per_step": q_bytes},
           "time_split_ms": {"quant": q_ms, "gemm": g_ms, "step": ms_step},
           "per_site": per_site,
           "gpu_launches": args.steps * nS * 2,
           "clocks": clk.summary()}
    tr = traffic_from_profiles()
    if tr:
        out["roofline"]["traffic"] = tr.get("gemm_bytes_per_launch")
        out["roofline"]["traffic_note"] = "profiles/ncu_traffic.json (committed ncu capture); algorithmic " \
            f"{tr.get('gemm_algorithmic_bytes_per_launch', 0):.3g} B per launch"
        out["quantize"]["traffic"] = tr.get("quant_bytes_per_launch")

    # decode-size step (BASELINE configs[1] decode M): the same 4 sites at M=16 tokens, CUDA-graph
    # replay; the weights (~128 MB for the 4 sites, > L2) stream from HBM every step.  Default =
    # arc_linear (quantize kernel + split-K GEMM + reduce kernel); the one-kernel fused decode
    # linear (quantize + stream-K GEMM + fixed-order reduction) beside it.
    if not args.no_decode and world == 1:
        Md = 16
        xd = [synth.activation(Md, s.K, synth.Structure(s.K, 8, seed=5), seed=9, device=device) for s in sites]
        yd = [torch.empty(Md, s.N, dtype=torch.bfloat16, device=device) for s in sites]
        wsd = [A.Workspace(device) for _ in sites]
        dec = {}
        for mode in ("fused", "unfused"):
            for s, x_, y_, w_ in zip(sites, xd, yd, wsd):
                A.linear(x_, s.prof, s.qw, out=y_, ws=w_, mode=mode)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            gs_ = torch.cuda.Stream()
            with torch.cuda.stream(gs_):
                with torch.cuda.graph(g, stream=gs_):
                    for s, x_, y_, w_ in zip(sites, xd, yd, wsd):
                        A.linear(x_, s.prof, s.qw, out=y_, ws=w_, mode=mode)
            torch.cuda.synchronize()
            for _ in range(3):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 50
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            dec[mode] = e0.elapsed_time(e1) / reps
            del g
        dms = dec["unfused"]
        wbytes = sum(s.N * s.Kp * 9 // 16 for s in sites)
        dbytes = wbytes + sum(Md * s.K * 2 + Md * s.N * 2 for s in sites)
        out["decode"] = {"M_tokens": Md, "us_per_layer_step": dms * 1e3, "tflops": sum(2.0 * Md * s.N * (s.K + s.S)
                         for s in sites) / (dms * 1e-3) / 1e12,
                         "bytes_per_step": dbytes, "achieved_gbs": dbytes / (dms * 1e-3) / 1e9,
                         "hbm_frac": dbytes / (dms * 1e-3) / 1e9 / peaks["hbm"],
                         "fused_us_per_layer_step": dec["fused"] * 1e3,
                         "fused_hbm_frac": dbytes / (dec["fused"] * 1e-3) / 1e9 / peaks["hbm"],
                         "note": "4 sites x (quantize + split-K GEMM + reduce, PDL-chained) per step in one CUDA "
                                 "graph (arc_linear default); fused_* = the one-kernel fused decode linear "
                                 "(ARC_LINEAR_FUSED: quantize phase + grid barrier + stream-K GEMM + in-kernel "
                                 "reduction); bound = weight bytes / HBM"}

    # e2e through the public C-ABI host-buffer call (H2D of x and D2H of y inside the timed region)
    if not args.no_e2e:
        xs = [s.x.cpu().pin_memory() for s in sites]
        ys = [torch.empty(s.M, s.N, dtype=torch.bfloat16).pin_memory() for s in sites]
        wss = [torch.zeros(A.linear_hostio_workspace_size(s.M, s.qw), dtype=torch.uint8, device=device)
               for s in sites]
        for _ in range(2):
            for s, xh, yh, ws in zip(sites, xs, ys, wss):
                A.linear_hostio(xh, s.prof, s.qw, yh, ws)
        if pg is not None:
            torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        nE = max(1, min(args.steps, 5))
        for _ in range(nE):
            for s, xh, yh, ws in zip(sites, xs, ys, wss):
                A.linear_hostio(xh, s.prof, s.qw, yh, ws)
                if s.mode == "row" and pg is not None:
                    pass  # host-buffer variant reports the per-rank partial; reduction is the device path's
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / nE
        if pg is not None:
            t = torch.tensor([ems], dtype=torch.float64, device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = t.item()
        out["e2e"] = {"value": flops_job / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
                      "h2d_bytes_per_step": sum(x.numel() * 2 for x in xs),
                      "d2h_bytes_per_step": sum(y.numel() * 2 for y in ys),
                      "ms_per_step": ems, "api": "arc_linear_hostio (C-ABI, pinned host buffers)"}

    if rank == 0 and not args.no_cpu_baseline:
        meta = sites_meta_for_oracle(sites, 2)
        v, desc, secs = oracle_sample(meta, budget_s=25.0)
        out["cpu_baseline"] = {"value": v, "unit": "TFLOP/s", "cores": 1, "kind": "oracle",
                               "sample": f"2 rows per site x full N (quantize + exact int64 GEMM): {desc}; {secs:.1f}s"}
    if rank == 0:
        print(json.dumps(out))
    if pg is not None:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
