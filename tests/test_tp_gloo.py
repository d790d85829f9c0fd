"""Tensor-parallel host logic (paper_2601_07475_b200.tp) at world_size 2 with the gloo
backend on CPU; the compute is the oracle stand-in (tests/_oracle_backend.py).

Column-parallel: the concatenated shards equal the per-shard oracle linear.
Row-parallel: the all-reduced output equals sum_r oracle_linear(X_r, W_r) with
per-rank calibration, within the summed north_star bounds."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

M, K, N, S_INJ = 8, 256, 64, 16


def _inputs():
    from paper_2601_07475_b200 import synth
    st = synth.Structure(K, S_INJ, seed=0)
    x = synth.activation(M, K, st, seed=1)
    cal = synth.activation(256, K, st, seed=1000)
    w = synth.weight(N, K, seed=2)
    return x, cal, w


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_07475_b200 import tp
    from _oracle_backend import OracleBackend
    be = OracleBackend()
    x, cal, w = _inputs()
    # column-parallel: replicated input, same profile everywhere
    prof = be.calibrate([cal])
    col = tp.ColumnParallelLinear(w, prof, rank, world, backend=be)
    y_col = col.forward(x, out_dtype=torch.float64)
    # row-parallel: input sliced over K, per-rank calibration, all-reduce of the partials
    row = tp.RowParallelLinear(w, cal, rank, world, backend=be)
    lo, hi = row.shard.lo, row.shard.hi
    y_row = row.forward(x[:, lo:hi].contiguous(), out_dtype=torch.float64)
    # the all-reduce fused into the GEMM epilogue (symmetric output buffer): the same sum
    y_fused = row.forward(x[:, lo:hi].contiguous(), reduce="fused").clone()
    y_fused2 = row.forward(x[:, lo:hi].contiguous(), reduce="fused").clone()  # buffer re-zeroed per call
    np.save(os.path.join(outdir, f"fused{rank}.npy"), np.stack([y_fused.numpy(), y_fused2.numpy()]))
    np.save(os.path.join(outdir, f"col{rank}.npy"), y_col.numpy())
    np.save(os.path.join(outdir, f"row{rank}.npy"), y_row.numpy())
    np.save(os.path.join(outdir, f"S{rank}.npy"), np.array([row.profile.S]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_tp_world2_gloo():
    sys.path.insert(0, HERE)
    from paper_2601_07475_b200 import tp
    from _oracle_backend import OracleBackend
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        be = OracleBackend()
        x, cal, w = _inputs()
        # column-parallel reference: per-shard oracle with the shared profile
        prof = be.calibrate([cal])
        for r in range(world):
            lo, hi = tp.shard_range(N, r, world, align=8)
            qw = be.quantize_weight(w[lo:hi].contiguous(), prof)
            ref, _ = be.linear_bound(x, prof, qw)
            assert np.array_equal(np.load(os.path.join(d, f"col{r}.npy")), ref)
        # row-parallel reference: sum over ranks of the per-slice oracle (float64)
        ref = np.zeros((M, N))
        bound = np.zeros((M, N))
        for r in range(world):
            lo, hi = tp.shard_range(K, r, world, align=16)
            p = be.calibrate([cal[:, lo:hi].contiguous()])
            assert int(np.load(os.path.join(d, f"S{r}.npy"))[0]) == p.S
            qw = be.quantize_weight(w[:, lo:hi].contiguous(), p)
            y, b = be.linear_bound(x[:, lo:hi].contiguous(), p, qw)
            ref += y
            bound += b
        for r in range(world):
            got = np.load(os.path.join(d, f"row{r}.npy"))
            assert np.all(np.abs(got - ref) <= bound + 1e-12)
            fused = np.load(os.path.join(d, f"fused{r}.npy"))
            assert np.array_equal(fused[0], got) and np.array_equal(fused[1], got)


def test_shard_range():
    from paper_2601_07475_b200 import tp
    assert tp.shard_range(4096, 3, 8) == (1536, 2048)
    with pytest.raises(ValueError):
        tp.shard_range(4096 + 16, 0, 8)


# ----------------------------------------------------------------------------- sequence parallel (f2)
MS = 256  # 128 token rows per rank at world 2


def _sp_inputs():
    from paper_2601_07475_b200 import synth
    st = synth.Structure(K, S_INJ, seed=3)
    x = synth.activation(MS, K, st, seed=4)
    cal = synth.activation(256, K, st, seed=1001)
    w = synth.weight(N, K, seed=5)
    gamma = synth.rmsnorm_weight(K, seed=6)
    return x, cal, w, gamma


def _sp_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_07475_b200 import tp
    from _oracle_backend import OracleBackend
    be = OracleBackend()
    x, cal, w, gamma = _sp_inputs()
    rows = slice(rank * MS // world, (rank + 1) * MS // world)
    prof = be.calibrate([cal])
    sp = tp.SequenceParallelColumnLinear(w, prof, rank, world, backend=be)
    codes, sf = sp.gather_quantized(x[rows].contiguous())
    y = sp.forward(x[rows].contiguous(), out_dtype=torch.float64)
    yn = sp.forward(x[rows].contiguous(), gamma=gamma, eps=1e-5, out_dtype=torch.float64)
    # row-parallel with the sequence-parallel reduce-scatter
    row = tp.RowParallelLinear(w, cal, rank, world, backend=be)
    xs = x[:, row.shard.lo:row.shard.hi].contiguous()
    y_all = row.forward(xs, out_dtype=torch.float64, reduce="all")
    y_sc = row.forward(xs, out_dtype=torch.float64, reduce="scatter")
    for name, t in (("codes", codes), ("sf", sf), ("y", y), ("yn", yn), ("yall", y_all), ("ysc", y_sc)):
        np.save(os.path.join(outdir, f"sp_{name}{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sequence_parallel_world2_gloo():
    """each rank quantizes its M/P token rows (plain or RMSNorm-fused) and all-gathers the
    packed codes + scales: bit-identical to quantizing all M rows, so each rank's N-shard output equals
    the oracle's column-parallel shard exactly; the reduce-scatter variant of the row-parallel layer
    gives every rank its rows of the all-reduce result."""
    sys.path.insert(0, HERE)
    import oracle
    from paper_2601_07475_b200 import tp
    from _oracle_backend import OracleBackend
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_sp_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        be = OracleBackend()
        x, cal, w, gamma = _sp_inputs()
        prof = be.calibrate([cal])
        ac, asf = oracle.quantize_activation(oracle.as_bf16_bits(x), prof.perm, prof.S, prof.gs, prof.layout)
        xn = oracle.rmsnorm(oracle.as_bf16_bits(x), oracle.as_bf16_bits(gamma), 1e-5)
        nc, nsf = oracle.quantize_activation(xn, prof.perm, prof.S, prof.gs, prof.layout)
        for r in range(world):
            assert np.array_equal(np.load(os.path.join(d, f"sp_codes{r}.npy")), ac)
            assert np.array_equal(np.load(os.path.join(d, f"sp_sf{r}.npy")).reshape(-1), asf.reshape(-1))
            lo, hi = tp.shard_range(N, r, world, align=8)
            qw = be.quantize_weight(w[lo:hi].contiguous(), prof)
            ref, _ = oracle.gemm_reference(ac, asf, qw.codes, qw.sf, prof.gs, qw.gs)
            assert np.array_equal(np.load(os.path.join(d, f"sp_y{r}.npy")), ref)
            refn, _ = oracle.gemm_reference(nc, nsf, qw.codes, qw.sf, prof.gs, qw.gs)
            assert np.array_equal(np.load(os.path.join(d, f"sp_yn{r}.npy")), refn)
            y_all = np.load(os.path.join(d, f"sp_yall{r}.npy"))
            y_sc = np.load(os.path.join(d, f"sp_ysc{r}.npy"))
            assert np.array_equal(y_sc, y_all[r * MS // world:(r + 1) * MS // world])
