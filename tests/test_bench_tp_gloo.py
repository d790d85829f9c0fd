"""bench.py's tensor-parallel step (bench.build_sites / bench.run_step, the code the driver times at
N > 1) at world_size 2 over gloo on CPU, with the oracle stand-in as the compute backend: every
column-parallel site's output equals the oracle on its N shard with the shared profile, every
row-parallel site's all-reduced output equals the sum over ranks of the per-slice oracle linears
(per-rank calibration on balanced outliers, S_r = max(16, S/P)) within the summed north_star bounds,
and the per-rank S_r are what the bench reports."""
import os
import socket
import sys
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

M, S = 8, 32
SITES = [("qkv", 256, 96), ("o", 256, 64), ("gate_up", 256, 128), ("down", 512, 64)]
CAL = 256


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from _oracle_backend import BenchOracleBackend
    B = BenchOracleBackend()
    sites = bench.build_sites(B, M, rank, world, "cpu", "mp", out_dtype=torch.float64, S=S, cal_rows=CAL,
                              sites=SITES)
    bench.run_step(B, sites, pg=dist.group.WORLD)
    for s in sites:
        np.save(os.path.join(outdir, f"{s.name}{rank}.npy"), s.y.numpy())
    # the row-parallel reduction fused into the GEMM epilogue (symmetric output) gives the same sums
    bench.run_step(B, sites, pg=dist.group.WORLD, tp_reduce="fused")
    for s in sites:
        if s.mode == "row":
            np.save(os.path.join(outdir, f"{s.name}_fused{rank}.npy"), s.y_out.numpy())
        np.save(os.path.join(outdir, f"{s.name}_S{rank}.npy"), np.array([s.S, s.K, s.N]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_tp_step_world2_gloo():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    import zlib
    import bench
    from _oracle_backend import OracleBackend
    from paper_2601_07475_b200 import synth, tp
    world = 2
    be = OracleBackend()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for name, K, N in SITES:
            seed = zlib.crc32(name.encode()) % 1000
            row = name not in bench.COL_SITES
            st = synth.Structure(K, S, seed=seed * 31, shards=world if row else 1)
            cal = synth.activation(CAL, K, st, seed=seed + 1000)
            w = synth.weight(N, K, seed=seed * 7)
            x = synth.activation(M, K, st, seed=seed + 1)
            if not row:
                prof = be.calibrate([cal], s_override=S)
                for r in range(world):
                    lo, hi = tp.shard_range(N, r, world, align=8)
                    ref, _ = be.linear_bound(x, prof, be.quantize_weight(w[lo:hi].contiguous(), prof))
                    assert np.array_equal(np.load(os.path.join(d, f"{name}{r}.npy")), ref), name
                continue
            S_r = max(16, (S // world + 15) // 16 * 16)
            ref = np.zeros((M, N))
            bound = np.zeros((M, N))
            for r in range(world):
                lo, hi = tp.shard_range(K, r, world, align=16)
                # balanced injection: each K shard holds S / P outlier channels
                assert ((st.idx >= lo) & (st.idx < hi)).sum() == S // world
                p = be.calibrate([cal[:, lo:hi].contiguous()], s_override=S_r)
                got_S, got_K, got_N = np.load(os.path.join(d, f"{name}_S{r}.npy"))
                assert (got_S, got_K, got_N) == (S_r, K // world, N)
                y, b = be.linear_bound(x[:, lo:hi].contiguous(), p, be.quantize_weight(w[:, lo:hi].contiguous(), p))
                ref += y
                bound += b
            for r in range(world):
                got = np.load(os.path.join(d, f"{name}{r}.npy"))
                assert np.all(np.abs(got - ref) <= bound + 1e-12), name
                assert np.array_equal(np.load(os.path.join(d, f"{name}_fused{r}.npy")), got), name


def test_bench_gpus_n_fails_loudly_without_n_gpus():
    """`bench.py --gpus N` self-launches N ranks; with fewer than N visible GPUs it must exit non-zero
    instead of silently timing one GPU."""
    import subprocess
    if torch.cuda.device_count() >= 2:
        return
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "CUDA device(s) visible" in r.stderr
