#!/usr/bin/env python
"""Benchmark of the ARC-NVFP4 linear hot path on B200 (BASELINE.json metric:
"ARC NVFP4 linear TFLOPS (% FP4 tensor peak) + quantize HBM GB/s, 1/2/4/8 GPU").

One step = the four ARC linear sites of one decoder layer, each = arc_quantize_activation +
arc_gemm (what arc_linear runs), synthetic activations with injected outlier channels and random
weights:

* N = 1 (default workload llama3-8b, BASELINE configs[1], prefill M = 8192): fused qkv
  (K=4096 -> N=6144), o (4096 -> 4096), fused gate-up (4096 -> 28672), down (14336 -> 4096),
  S = 128 augmented channels each.
* N > 1 (default workload llama3-70b, BASELINE configs[3]): Megatron tensor parallelism of one
  LLaMA-3-70B layer (strong scaling): qkv (8192 -> 10240) and gate-up (8192 -> 57344)
  column-parallel over N (replicated input, no communication), o (8192 -> 8192) and down
  (28672 -> 8192) row-parallel over K with per-rank calibration (S_r = max(16, 128/P), outliers
  injected balanced over the K shards) and an NCCL all-reduce of Y.  `--workload llama3-70b` at
  N = 1 gives the same layer unsharded.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl arc|reference] [--M 8192]
                    [--workload auto|llama3-8b|llama3-70b] [--tp-layout mp|sp]

`--gpus N` with N > 1 and no WORLD_SIZE in the environment re-executes itself under
torch.distributed.run with N ranks (one per GPU); it exits non-zero if fewer than N GPUs are visible.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time
import zlib

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2601_07475_b200 import synth  # noqa: E402

S_AUG = 128
COL_SITES = ("qkv", "gate_up")
WORKLOADS = {
    "llama3-8b": (synth.LLAMA3_8B_SITES, "llama3-8b-layer-4-arc-linears-prefill"),
    "llama3-70b": (synth.LLAMA3_70B_SITES, "llama3-70b-layer-4-arc-linears-tp"),
}
CAL_ROWS = 4096


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


def _gs_float(g) -> float:
    return float(g.item()) if isinstance(g, torch.Tensor) else float(g)


# ----------------------------------------------------------------------------- workload
class Site:
    """One ARC linear site of the layer on this rank.  mode: 'full' (1 GPU), 'col' (column-parallel
    shard of N) or 'row' (row-parallel shard of K).  Sharded sites are built with
    paper_2601_07475_b200.tp (the tested host logic).  layout 'sp' (sequence parallel): a
    col site quantizes its M/P token rows and all-gathers the packed codes + scales; a row site
    reduce-scatters its output over tokens.  'mp': col sites quantize the replicated M rows, row sites
    all-reduce.  B is the compute backend (the libarc binding; tests pass an oracle stand-in)."""

    def __init__(self, B, name, K, N, M, S, rank, world, device, layout="mp", out_dtype=torch.bfloat16,
                 cal_rows=CAL_ROWS, keep_host=False):
        from paper_2601_07475_b200 import tp
        self.name, self.M = name, M
        self.mode = "full" if world == 1 else ("col" if name in COL_SITES else "row")
        self.sp = layout == "sp" and world > 1
        self.world, self.rank = world, rank
        seed = zlib.crc32(name.encode()) % 1000
        st = synth.Structure(K, S, seed=seed * 31, shards=world if self.mode == "row" else 1)
        cal = synth.activation(cal_rows, K, st, seed=seed + 1000, device=device)
        w = synth.weight(N, K, seed=seed * 7, device=device)
        x = synth.activation(M, K, st, seed=seed + 1, device=device)
        self.S_target = S
        if self.mode == "full":
            self.prof = B.calibrate([cal], s_override=S)
            self.qw = B.quantize_weight(w, self.prof)
            self.x, self.w_local, self.cal_local = x, w, cal
        elif self.mode == "col":
            prof = B.calibrate([cal], s_override=S)
            lin = tp.ColumnParallelLinear(w, prof, rank, world, backend=B)
            self.prof, self.qw, self.x = lin.profile, lin.qweight, x
            self.w_local = w[lin.shard.lo:lin.shard.hi]
            self.cal_local = cal
        else:
            S_r = max(16, (S // world + 15) // 16 * 16)
            lin = tp.RowParallelLinear(w, cal, rank, world, s_override=S_r, backend=B)
            self.lin = lin
            self.prof, self.qw = lin.profile, lin.qweight
            self.x = x[:, lin.shard.lo:lin.shard.hi].contiguous()
            self.w_local = w[:, lin.shard.lo:lin.shard.hi]
            self.cal_local = cal[:, lin.shard.lo:lin.shard.hi]
        if not keep_host:
            self.w_local = self.cal_local = None
        del cal, w, x
        Kl, Nl, S_l = self.x.shape[1], self.qw.codes.shape[0], self.prof.S
        self.K, self.N, self.S = Kl, Nl, S_l
        Kp, cb, sb = B.buffer_sizes(M, Kl, S_l)
        self.Kp = Kp
        self.codes = torch.empty(M, Kp // 2, dtype=torch.uint8, device=device)
        self.sf = torch.empty(sb, dtype=torch.uint8, device=device)
        self.y = torch.empty(M, Nl, dtype=out_dtype, device=device)
        self.m_q = M  # rows this rank quantizes
        self.out_rows = M // world if (self.sp and self.mode == "row") else M
        if self.sp and self.mode == "col":
            ml = M // world
            assert ml % 128 == 0, "sequence-parallel rows per rank must be a multiple of 128"
            self.x = self.x[rank * ml:(rank + 1) * ml].contiguous()
            self.m_q = ml
        self.ws = B.Workspace(device)
        self.flops = 2.0 * M * Nl * (Kl + S_l)                       # SPEC S:322 cost model, algorithmic
        self.flops_eff = 2.0 * M * Nl * Kl
        self.q_bytes = self.m_q * (2 * Kl + Kp // 2 + Kp // 16) + 4 * Kl  # bf16 read + codes + scales + perm
        self.g_bytes = Nl * Kp * 9 // 16 + M * Kp * 9 // 16 + M * Nl * 2
        self.comm_bytes = M * Nl * self.y.element_size() if self.mode == "row" else (
            M * (Kp // 2 + Kp // 16) if self.sp else 0)


def workload_sites(name):
    return WORKLOADS[name][0]


def build_sites(B, M, rank, world, device, layout="mp", workload="llama3-8b", out_dtype=torch.bfloat16,
                S=S_AUG, cal_rows=CAL_ROWS, keep_host=False, sites=None):
    out = []
    for name, K, N in (sites or workload_sites(workload)):
        out.append(Site(B, name, K, N, M, S, rank, world, device, layout, out_dtype, cal_rows, keep_host))
    return out


def run_step(B, sites, ev=None, pg=None, tp_reduce="nccl"):
    """One pass of the layer's linears on this rank.  ev[i] = 4 CUDA events per site: before quantize,
    after quantize, after GEMM, after the collective.  tp_reduce "fused": row-parallel sites add their
    partials into every rank's symmetric-memory output from the GEMM epilogue (arc_gemm_reduce, NVLS
    multicast or P2P) instead of an NCCL all-reduce; their quantize + GEMM + reduction is timed as
    "gemm"."""
    from paper_2601_07475_b200 import tp
    for i, s in enumerate(sites):
        if ev is not None:
            ev[i][0].record()
        if tp_reduce == "fused" and s.mode == "row" and pg is not None and not s.sp:
            if ev is not None:
                ev[i][1].record()
            s.y_out = s.lin.forward(s.x, reduce="fused")
            if ev is not None:
                ev[i][2].record()
                ev[i][3].record()
            continue
        if s.sp and s.mode == "col":
            # sequence parallel: quantize this rank's token rows, all-gather the packed codes + scales
            c_loc, sf_loc = B.quantize_activation(s.x, s.prof)
            s.codes.copy_(tp._all_gather_rows(c_loc, pg))
            s.sf.copy_(tp._all_gather_rows(sf_loc.reshape(s.m_q // 128, -1), pg).reshape(-1))
        else:
            B.quantize_activation(s.x, s.prof, s.codes, s.sf)
        if ev is not None:
            ev[i][1].record()
        B.gemm(s.codes, s.sf, s.prof.gs, s.qw, out=s.y, ws=s.ws)
        if ev is not None:
            ev[i][2].record()
        if s.mode == "row" and pg is not None:
            if s.sp:
                s.y_out = tp._reduce_scatter_rows(s.y, pg)
            else:
                torch.distributed.all_reduce(s.y, group=pg)
        if ev is not None:
            ev[i][3].record()


# ----------------------------------------------------------------------------- oracle (CPU) legs
def lscpu_model():
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_site(name, K, N, S, rows, cal_rows=CAL_ROWS):
    """Everything the oracle needs for one site, made by the oracle alone on the host: seeded CPU
    synthetic data of the workload's shapes, calibration (abs-max + outlier selection), the weight's
    tensor scale and its ARC quantization (outlier blocks duplicated).  Untimed (offline work)."""
    import oracle
    seed = zlib.crc32(name.encode()) % 1000
    st = synth.Structure(K, S, seed=seed * 31)
    cal = oracle.as_bf16_bits(synth.activation(cal_rows, K, st, seed=seed + 1000))
    w = synth.weight(N, K, seed=seed * 7)
    gs_w = oracle.tensor_scale(float(w.float().abs().max()))
    wb = oracle.as_bf16_bits(w)
    del w
    x = oracle.as_bf16_bits(synth.activation(rows, K, st, seed=seed + 1))
    sel = oracle.select_outliers(oracle.calib_absmax(cal), S)
    with oracle.openmp():
        wc, wsf = oracle.quantize_weight(wb, sel["perm"], sel["S"], gs_w)
    return dict(name=name, K=K, N=N, S=sel["S"], x=x, perm=sel["perm"], gs=sel["gs"], wc=wc, wsf=wsf, gs_w=gs_w)


def oracle_step(meta, openmp=True):
    """One bounded sample of the workload on the oracle: ARC-quantize each site's sample rows and run
    the exact GEMM of those rows against the site's full weight.  Returns (flops, seconds)."""
    import oracle
    ctx = oracle.openmp() if openmp else _Null()
    flops, t0 = 0.0, time.perf_counter()
    with ctx:
        for m in meta:
            ac, asf = oracle.quantize_activation(m["x"], m["perm"], m["S"], m["gs"])
            oracle.gemm_exact(ac, asf, m["wc"], m["wsf"])
            flops += 2.0 * m["x"].shape[0] * m["N"] * (m["K"] + m["S"])
    return flops, time.perf_counter() - t0


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def oracle_meta_from_sites(sites, rows):
    """Oracle-side preparation from the bench's own site inputs (the same bf16 activations, calibration
    rows and weights, copied to the host): the oracle calibrates and quantizes the weights itself --
    nothing produced by libarc is used."""
    import oracle
    meta = []
    for s in sites:
        cal = oracle.as_bf16_bits(s.cal_local.cpu())
        w = s.w_local.cpu()
        gs_w = oracle.tensor_scale(float(w.float().abs().max()))
        sel = oracle.select_outliers(oracle.calib_absmax(cal), s.S)
        with oracle.openmp():
            wc, wsf = oracle.quantize_weight(oracle.as_bf16_bits(w), sel["perm"], sel["S"], gs_w)
        meta.append(dict(name=s.name, K=s.K, N=s.N, S=sel["S"], x=oracle.as_bf16_bits(s.x[:rows].cpu()),
                         perm=sel["perm"], gs=sel["gs"], wc=wc, wsf=wsf, gs_w=gs_w))
    return meta


def parity_sample(sites, meta):
    """The timed GPU step's outputs on the sampled rows against the oracle's exact GEMM (north_star
    bound 1e-5 * sum|ab| + the bf16 rounding of the stored output)."""
    import oracle
    out = {}
    for s, m in zip(sites, meta):
        rows = m["x"].shape[0]
        with oracle.openmp():
            ac, asf = oracle.quantize_activation(m["x"], m["perm"], m["S"], m["gs"])
            yref, bound = oracle.gemm_reference(ac, asf, m["wc"], m["wsf"], m["gs"], m["gs_w"])
        y = s.y[:rows].float().cpu().numpy().astype(np.float64)
        tol = bound + np.abs(yref) * 2.0 ** -8
        out[s.name] = {"rows": rows, "max_err_over_bound": float(np.max(np.abs(y - yref) / np.maximum(tol, 1e-300))),
                       "ok": bool(np.all(np.abs(y - yref) <= tol))}
    return out


# ----------------------------------------------------------------------------- GPU side legs
def time_graph(fn, reps=50, warm=3):
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.synchronize()
    for _ in range(warm):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def decode_sweep(A, sites, device, peaks, Ms=(1, 4, 16, 32, 64)):
    """BASELINE configs[1] decode token counts: the same 4 sites at M tokens, CUDA-graph replay.  The
    weights of the 4 sites (~128 MB at LLaMA-3-8B, > L2) stream from HBM every step.  Bound = weight
    + activation bytes / HBM.  Default arc_linear (per site: the direct-gather quantize kernel + the
    cluster split-K GEMM whose K partials are reduced in distributed shared memory, decode_gemm.cu) and,
    beside it, ARC_LINEAR_FUSED (one in-kernel-quantize stream-K kernel per site)."""
    out = []
    wbytes = sum(s.N * s.Kp * 9 // 16 for s in sites)
    for Md in Ms:
        xd = [synth.activation(Md, s.K, synth.Structure(s.K, 8, seed=5), seed=9, device=device) for s in sites]
        yd = [torch.empty(Md, s.N, dtype=torch.bfloat16, device=device) for s in sites]
        wsd = [A.Workspace(device) for _ in sites]

        def step():
            for s, x_, y_, w_ in zip(sites, xd, yd, wsd):
                A.linear(x_, s.prof, s.qw, out=y_, ws=w_)
        ms = time_graph(step)

        def step_fused():
            for s, x_, y_, w_ in zip(sites, xd, yd, wsd):
                A.linear(x_, s.prof, s.qw, out=y_, ws=w_, mode="fused")
        ms_f = time_graph(step_fused)
        dbytes = wbytes + sum(Md * s.K * 2 + Md * s.N * 2 for s in sites)
        out.append({"M_tokens": Md, "us_per_layer_step": ms * 1e3, "bytes_per_step": dbytes,
                    "achieved_gbs": dbytes / (ms * 1e-3) / 1e9, "hbm_frac": dbytes / (ms * 1e-3) / 1e9 / peaks["hbm"],
                    "tflops": sum(2.0 * Md * s.N * (s.K + s.S) for s in sites) / (ms * 1e-3) / 1e12,
                    "fused_us_per_layer_step": ms_f * 1e3,
                    "fused_hbm_frac": dbytes / (ms_f * 1e-3) / 1e9 / peaks["hbm"]})
    return out


QWEN_SITES = {  # (site, K, N): BASELINE configs[2] (Qwen2.5-7B / 32B linear shapes)
    "qwen2.5-7b": [("qkv", 3584, 4608), ("down", 18944, 3584)],
    "qwen2.5-32b": [("qkv", 5120, 7168), ("down", 27648, 5120)],
}


def s_sweep(A, device, M=2048, Ss=(0, 64, 128, 256)):
    """BASELINE configs[2]: GEMM time vs the augmented channel count S on Qwen2.5-7B / 32B shapes (the
    paper's Fig.8a question): arc_gemm of the quantized operands, CUDA graph of 5 launches."""
    out = []
    for model, sites in QWEN_SITES.items():
        for site, K, N in sites:
            st = synth.Structure(K, 128, seed=K)
            x = synth.activation(M, K, st, seed=K + 1, device=device)
            w = synth.weight(N, K, seed=N, device=device)
            y = torch.empty(M, N, dtype=torch.bfloat16, device=device)
            base = A.calibrate([x[:1024]], s_override=0)
            perm = base.perm.cpu().numpy()
            rec = {"model": model, "site": site, "M": M, "K": K, "N": N, "by_S": []}
            for S in Ss:
                prof = A.profile_from(perm, S, float(base.gs.item()))
                qw = A.quantize_weight(w, prof)
                codes, sf = A.quantize_activation(x, prof)
                ms = time_graph(lambda: A.gemm(codes, sf, prof.gs, qw, out=y), reps=5)
                rec["by_S"].append({"S": S, "gemm_us": ms * 1e3, "tflops_K_plus_S": 2.0 * M * N * (K + S) / (ms * 1e-3) / 1e12})
                del qw, codes, sf
            t0 = rec["by_S"][0]["gemm_us"]
            for r in rec["by_S"]:
                r["time_vs_S0"] = r["gemm_us"] / t0
            out.append(rec)
            del x, w, y
            torch.cuda.empty_cache()
    return out


def layer_chain_config5():
    """BASELINE configs[4]: scripts/layer_chain.py (one LLaMA-3-8B decoder layer's linear chain with fused
    producers at 16 x 2048 tokens vs BF16 cuBLAS and plain NVFP4) in a subprocess; its JSON summary."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "layer_chain.py")], capture_output=True, text=True,
                       timeout=600)
    if r.returncode != 0:
        return {"error": (r.stderr or "")[-400:]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    return {"M_tokens": d["M_tokens"], "us": d["us"], "arc_speedup_vs_bf16": d["arc_speedup_vs_bf16"],
            "arc_vs_nvfp4_overhead": d["arc_vs_nvfp4_overhead"], "fusion_saving_vs_unfused": d["fusion_saving_vs_unfused"]}


def quantize_streaming(A, device, peaks, reps=5):
    """The quantize pass at streaming sizes (footprint >= 4x the 126 MB L2, so every launch reads its
    input from HBM): M=65536 x K=4096 and M=16384 x K=14336, S = 128."""
    out = []
    for M, K in ((65536, 4096), (16384, 14336)):
        st = synth.Structure(K, S_AUG, seed=K)
        x = synth.activation(M, K, st, seed=K + 1, device=device)
        prof = A.calibrate([synth.activation(1024, K, st, seed=K + 2, device=device)], s_override=S_AUG)
        codes, sf = A.quantize_activation(x, prof)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for e0, e1 in evs:
            e0.record()
            A.quantize_activation(x, prof, codes, sf)
            e1.record()
        torch.cuda.synchronize()
        us = float(np.median([e0.elapsed_time(e1) for e0, e1 in evs])) * 1e3
        Kp = codes.shape[1] * 2
        nbytes = M * (2 * K + Kp // 2 + Kp // 16) + 4 * K
        out.append({"M": M, "K": K, "S": S_AUG, "bytes": nbytes, "read_mb": M * K * 2 / 1e6, "us": us,
                    "achieved_gbs": nbytes / (us * 1e-6) / 1e9, "frac": nbytes / (us * 1e-6) / 1e9 / peaks["hbm"]})
        del x, codes, sf
    torch.cuda.empty_cache()
    return out


def nccl_lines(path):
    keep = []
    try:
        for ln in open(path):
            if any(k in ln for k in ("Init COMPLETE", "NVLS", "nvls", "CollNet", "comm 0x", "Using network",
                                     "P2P/CUMEM", "Connected all")):
                keep.append(ln.strip()[:240])
    except OSError:
        pass
    return keep[:40]


# ----------------------------------------------------------------------------- arms
def reference_arm(args, config, metric):
    """The oracle as the reference arm (there is no reference implementation to install:
    /root/reference holds only the paper and a spec).  Rank 0 only; self-contained: the oracle
    builds its own calibration and weights from seeded CPU data, libarc is never loaded."""
    import oracle
    oracle.build()
    rows = 1
    meta = [oracle_site(name, K, N, S_AUG, rows) for name, K, N in workload_sites(config["_workload"])]
    for _ in range(min(args.warmup, 1)):
        oracle_step(meta)
    flops, secs = 0.0, []
    for _ in range(args.steps):
        f, t = oracle_step(meta)
        flops = f
        secs.append(t)
    with oracle.openmp():
        cores = oracle.num_threads()
    v = flops / float(np.median(secs)) / 1e12
    cfg = {k: v_ for k, v_ in config.items() if not k.startswith("_")}
    sample = f"{rows} activation row per site x full N (quantize + exact int64 GEMM), unsharded layer: " + \
        ";".join(f"{m['name']}:{rows}x{m['N']}x{m['K']}+{m['S']}" for m in meta)
    line = {"impl": "reference", "metric": metric, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(secs)) * 1e3,
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "int64-exact (oracle)", "data": "synthetic (seeded, CPU)", "config": cfg,
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "nproc": os.cpu_count(), "cpu_model": lscpu_model()},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="arc", choices=["arc", "reference"])
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--workload", default="auto", choices=["auto"] + list(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-streaming", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the config-3 S sweep and the config-5 layer chain")
    ap.add_argument("--tp-reduce", default="nccl", choices=["nccl", "fused"],
                    help="N>1 row-parallel sites: NCCL all-reduce after the GEMM, or the reduction fused into the GEMM "
                         "epilogue over symmetric memory (NVLS multimem / P2P)")
    ap.add_argument("--tp-layout", default="mp", choices=["mp", "sp"],
                    help="N>1: sequence-parallel (quantize M/P rows + all-gather packed codes, reduce-scatter) "
                         "or plain Megatron (replicated quantize, all-reduce)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    in_dist = "WORLD_SIZE" in os.environ
    if args.impl == "arc" and args.gpus > 1 and not in_dist:
        n = torch.cuda.device_count()
        if n < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible")
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if in_dist and world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    workload = args.workload if args.workload != "auto" else ("llama3-8b" if args.gpus == 1 else "llama3-70b")
    metric = "ARC NVFP4 linear TFLOPS"
    config = {"workload": WORKLOADS[workload][1], "M_tokens": args.M, "S": S_AUG,
              "sites": [f"{n}:K{k}xN{nn}" for n, k, nn in workload_sites(workload)],
              "parallelism": "single" if args.gpus == 1 else f"tp{args.gpus}-{args.tp_layout}-{args.tp_reduce}",
              "l2": "per-step footprint > 4x L2 (no flush needed)", "_workload": workload}

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, config, metric)
        return

    pg = None
    nccl_log = None
    if world > 1:
        nccl_log = f"/tmp/arc_bench_nccl.{os.getpid()}.log"
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log)
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = torch.distributed.group.WORLD
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    peaks = _peaks()
    fp4_burst = peaks["bf16"] * 4.0     # guide's nominal fp4 / bf16 ratio (9 / 2.25)
    fp4_sus = peaks["bf16_sus"] * 4.0

    from paper_2601_07475_b200 import arc as A
    if not A.device_supported():
        raise SystemExit("bench.py: current device is not sm_100 -- the ARC path has no fallback")
    keep = rank == 0 and world == 1 and not args.no_cpu_baseline
    sites = build_sites(A, args.M, rank, world, device, args.tp_layout, workload, keep_host=keep)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        run_step(A, sites, pg=pg, tp_reduce=args.tp_reduce)
    torch.cuda.synchronize()

    nS = len(sites)
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(nS)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if pg is not None:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        start.record()
        for k in range(args.steps):
            run_step(A, sites, ev=evs[k], pg=pg, tp_reduce=args.tp_reduce)
        stop.record()
        torch.cuda.synchronize()
    if pg is not None:
        torch.distributed.barrier()
    ms = start.elapsed_time(stop)

    def seg(i, a, b):
        return sum(evs[k][i][a].elapsed_time(evs[k][i][b]) for k in range(args.steps)) / args.steps

    per_site = {}
    for i, s in enumerate(sites):
        per_site[s.name] = {"mode": s.mode, "K": s.K, "N": s.N, "S": s.S, "quant_us": 1e3 * seg(i, 0, 1),
                            "gemm_us": 1e3 * seg(i, 1, 2), "comm_us": 1e3 * seg(i, 2, 3)}
    q_ms = sum(v["quant_us"] for v in per_site.values()) / 1e3
    g_ms = sum(v["gemm_us"] for v in per_site.values()) / 1e3
    c_ms = sum(v["comm_us"] for v in per_site.values()) / 1e3
    if pg is not None:
        t = torch.tensor([ms, q_ms, g_ms, c_ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, q_ms, g_ms, c_ms = t.tolist()

    flops_rank = sum(s.flops for s in sites)
    flops_job = flops_rank * world        # TP shards one layer; each rank's flops are disjoint parts of it
    ms_step = ms / args.steps
    value = flops_job / (ms_step * 1e-3) / 1e12
    g_tflops = flops_rank / (g_ms * 1e-3) / 1e12
    q_bytes = sum(s.q_bytes for s in sites)
    q_gbs = q_bytes / (q_ms * 1e-3) / 1e9
    for s in sites:
        v = per_site[s.name]
        v["gemm_tflops"] = s.flops / (v["gemm_us"] * 1e-6) / 1e12
        v["gemm_frac_burst"] = v["gemm_tflops"] / fp4_burst
        v["quant_gbs"] = s.q_bytes / (v["quant_us"] * 1e-6) / 1e9
        v["quant_frac"] = v["quant_gbs"] / peaks["hbm"]
    clocks = clk.summary()
    power_capped = "sw_power_cap" in clocks.get("reasons", [])
    peak = fp4_burst  # the timed region is ~0.1 s at full clock: the burst peak (sustained reported beside)
    out = {"metric": metric, "value": value, "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
           "dtype": "nvfp4(e2m1+ue4m3)->fp32acc->bf16",
           "data": "synthetic (LLaMA-3 shapes, injected outlier channels, random weights)",
           "config": {k: v_ for k, v_ in config.items() if not k.startswith("_")},
           "roofline": {"bound": "tensor", "kernel": "arc_gemm_kernel (4 launches/step)",
                        "achieved": g_tflops, "peak": peak, "unit": "TFLOP/s", "frac": g_tflops / peak,
                        "peak_note": (f"{peaks['src']} bf16 burst {peaks['bf16']} x 4 (fp4/bf16 nominal 9/2.25); "
                                      f"{'sw_power_cap seen in a sample' if power_capped else 'no power cap seen'}"),
                        "frac_burst": g_tflops / fp4_burst, "frac_sustained": g_tflops / fp4_sus,
                        "frac_datasheet_9pf": g_tflops / 9000.0, "traffic": None},
           "quantize": {"bound": "hbm", "kernel": "arc_quant_kernel (4 launches/step)", "achieved": q_gbs,
                        "peak": peaks["hbm"], "unit": "GB/s", "frac": q_gbs / peaks["hbm"],
                        "bytes_per_step": q_bytes},
           "time_split_ms": {"quant": q_ms, "gemm": g_ms, "comm": c_ms, "step": ms_step},
           "per_site": per_site,
           "gpu_launches": args.steps * nS * 2,
           "clocks": clocks}
    tr = os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")
    if os.path.exists(tr):
        try:
            d = json.load(open(tr))
            out["roofline"]["traffic"] = d.get("gemm_bytes_per_launch")
            out["roofline"]["traffic_note"] = f"ncu --set full capture ({d.get('source', tr)}); algorithmic " \
                f"{d.get('gemm_algorithmic_bytes_per_launch', 0):.3g} B/launch; per-site: {d.get('per_site')}"
            out["quantize"]["traffic"] = d.get("quant_bytes_per_launch")
        except Exception:
            pass

    if world > 1:
        S_r = {}
        for s in sites:
            t = torch.tensor([s.S], dtype=torch.int64, device=device)
            allS = [torch.zeros_like(t) for _ in range(world)]
            torch.distributed.all_gather(allS, t)
            S_r[s.name] = [int(a.item()) for a in allS]
        tp_out = {"layout": args.tp_layout, "gemm_only_ms": q_ms + g_ms, "gemm_plus_comm_ms": ms_step,
                  "comm_ms": c_ms, "S_r_per_rank": S_r, "sites": {}}
        for s in sites:
            v = per_site[s.name]
            if s.mode == "row":
                bus = (2.0 if not s.sp else 1.0) * (world - 1) / world * s.comm_bytes / (v["comm_us"] * 1e-6) / 1e9
                tp_out["sites"][s.name] = {"collective": "reduce_scatter" if s.sp else "all_reduce",
                                           "bytes": s.comm_bytes, "us": v["comm_us"], "busbw_gbs": bus}
        out["tp"] = tp_out
        if rank == 0 and nccl_log:
            out["nccl"] = nccl_lines(nccl_log)

    if not args.no_decode and world == 1:
        out["decode"] = decode_sweep(A, sites, device, peaks)
    if not args.no_streaming and world == 1:
        out["quantize_streaming"] = quantize_streaming(A, device, peaks)
    if not args.no_extras and world == 1:
        out["config3_s_sweep"] = s_sweep(A, device)
        out["config5_layer_chain"] = layer_chain_config5()
        if workload == "llama3-8b":
            # the decode path on the LLaMA-3-70B layer's weights (488 MB per 4-site step, configs[3] shapes
            # unsharded): the fixed per-launch latencies that bound the 8B step are amortized there
            s70 = build_sites(A, 128, 0, 1, device, workload="llama3-70b", cal_rows=1024)
            out["decode_llama3_70b_layer"] = decode_sweep(A, s70, device, peaks, Ms=(1, 16, 64))
            del s70
            torch.cuda.empty_cache()

    # e2e through the public API: every step copies the step's inputs from pinned host memory to the
    # device and the outputs back (world 1: the C-ABI host-buffer call arc_linear_hostio does both
    # inside the call; TP: the same copies around the device path incl. its collectives)
    if not args.no_e2e:
        xs = [s.x.cpu().pin_memory() for s in sites]
        ys = [torch.empty(s.out_rows, s.N, dtype=s.y.dtype).pin_memory() for s in sites]
        if world == 1:
            wss = [torch.zeros(A.linear_hostio_workspace_size(s.M, s.qw), dtype=torch.uint8, device=device)
                   for s in sites]

            def e2e_step():
                # arc_linear_hostio_async per site (H2D / linear / D2H pipelined over row chunks, the copies
                # of consecutive sites overlapping), then one arc_linear_hostio_wait
                for s, xh, yh, ws in zip(sites, xs, ys, wss):
                    A.linear_hostio(xh, s.prof, s.qw, yh, ws, wait=False)
                A.linear_hostio_wait()
        else:
            def e2e_step():
                for s, xh in zip(sites, xs):
                    s.x.copy_(xh, non_blocking=True)
                run_step(A, sites, pg=pg, tp_reduce=args.tp_reduce)
                for s, yh in zip(sites, ys):
                    yh.copy_(s.y_out if (s.mode == "row" and hasattr(s, "y_out")) else s.y, non_blocking=True)
        for _ in range(2):
            e2e_step()
        if pg is not None:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        nE = max(1, min(args.steps, 5))
        for _ in range(nE):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / nE
        if pg is not None:
            t = torch.tensor([ems], dtype=torch.float64, device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = t.item()
        out["e2e"] = {"value": flops_job / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
                      "h2d_bytes_per_step": sum(x.numel() * x.element_size() for x in xs),
                      "d2h_bytes_per_step": sum(y.numel() * y.element_size() for y in ys),
                      "ms_per_step": ems,
                      "api": "arc_linear_hostio_async + arc_linear_hostio_wait (C-ABI, pinned host buffers)" if world == 1 else
                             "arc quantize+gemm per rank + NCCL collectives, pinned host copies in the step"}

    if keep:
        import oracle
        oracle.build()
        rows = 2
        run_step(A, sites)  # the outputs the parity sample compares
        torch.cuda.synchronize()
        meta = oracle_meta_from_sites(sites, rows)
        out["parity_sample"] = parity_sample(sites, meta)
        f1, t1 = oracle_step(meta, openmp=False)
        fN, tN = oracle_step(meta, openmp=True)
        with oracle.openmp():
            cores = oracle.num_threads()
        desc = ";".join(f"{m['name']}:{rows}x{m['N']}x{m['K']}+{m['S']}" for m in meta)
        out["cpu_baseline"] = {"value": fN / tN / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                               "sample": f"{rows} rows per site x full N (quantize + exact int64 GEMM), "
                                         f"OpenMP over output columns: {desc}; {tN:.2f} s",
                               "single_thread_value": f1 / t1 / 1e12, "single_thread_s": t1,
                               "nproc": os.cpu_count(), "cpu_model": lscpu_model(),
                               "prep": "oracle's own calibration + weight quantization of the same bf16 inputs"}
    if rank == 0:
        print(json.dumps(out))
    if pg is not None:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
