"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds none of the method's arithmetic: it only draws random numbers
with the structure of the paper's workloads:
a few persistent high-magnitude outlier channels (Fig.2) on a
Gaussian bulk with a per-token magnitude spread, rounded to bf16 (RNE).

recipe:
  structure(K, S_inj, seed): idx = S_inj distinct channels, gain ~ logU[32, 128]
  activation(M, K, st, seed): X = N(0,1) * exp(0.5 N(0,1))[row] ; X[:, idx] *= gain
  weight(N, K, seed): N(0,1) / sqrt(K)
  rmsnorm_weight(K, seed): exp(0.3 N(0,1))  (positive per-channel RMSNorm gains around 1)
  gate_up(M, K, st, seed): bf16 [M, 2K] = [gate | up] with gate = 2 N(0,1) (pre-activation spread
      that covers SiLU's negative lobe and linear tail) and up = activation(M, K, st) (the
      down-proj input's outlier channels, Fig.2, come through the up half)
"""
from __future__ import annotations

import math
import numpy as np
import torch


class Structure:
    def __init__(self, K: int, S_inj: int, seed: int = 0, shards: int = 1):
        """shards > 1: S_inj / shards channels inside each of `shards` contiguous K slices (the balanced
        outliers of a row-parallel layer, SURVEY.md §8(e) "Outlier balance")."""
        rng = np.random.default_rng(seed)
        self.K = K
        if shards > 1:
            ks, per = K // shards, max(1, S_inj // shards)
            self.idx = np.sort(np.concatenate([r * ks + rng.choice(ks, per, replace=False)
                                               for r in range(shards)])).astype(np.int64)
        else:
            self.idx = np.sort(rng.choice(K, S_inj, replace=False)).astype(np.int64)
        self.gain = np.exp(rng.uniform(math.log(32.0), math.log(128.0), self.idx.size)).astype(np.float32)


def activation(M: int, K: int, st: Structure, seed: int, device="cpu") -> torch.Tensor:
    """bf16 [M, K] activation with injected outlier channels."""
    g = torch.Generator(device=device).manual_seed(int(seed))
    row = torch.exp(0.5 * torch.randn(M, generator=g, device=device, dtype=torch.float32))
    x = torch.randn(M, K, generator=g, device=device, dtype=torch.float32) * row[:, None]
    if st.idx.size:
        idx = torch.as_tensor(st.idx, device=device)
        x[:, idx] *= torch.as_tensor(st.gain, device=device)
    return x.to(torch.bfloat16)


def weight(N: int, K: int, seed: int, device="cpu") -> torch.Tensor:
    g = torch.Generator(device=device).manual_seed(int(seed) + 7919)
    w = torch.randn(N, K, generator=g, device=device, dtype=torch.float32) / math.sqrt(K)
    return w.to(torch.bfloat16)


def rmsnorm_weight(K: int, seed: int, device="cpu") -> torch.Tensor:
    """bf16 [K] RMSNorm gain vector (the gamma of the attention / MLP input norms)."""
    g = torch.Generator(device=device).manual_seed(int(seed) + 104729)
    return torch.exp(0.3 * torch.randn(K, generator=g, device=device, dtype=torch.float32)).to(torch.bfloat16)


def gate_up(M: int, K: int, st: Structure, seed: int, device="cpu") -> torch.Tensor:
    """bf16 [M, 2K] fused gate_up output: gate in columns [0, K), up in [K, 2K)."""
    g = torch.Generator(device=device).manual_seed(int(seed) + 15485863)
    gate = 2.0 * torch.randn(M, K, generator=g, device=device, dtype=torch.float32)
    up = activation(M, K, st, seed, device=device).float()
    return torch.cat([gate, up], dim=1).to(torch.bfloat16)


def random_perm(K: int, seed: int) -> np.ndarray:
    """A seeded permutation (used where a test wants an arbitrary valid perm)."""
    return np.random.default_rng(seed).permutation(K).astype(np.int32)


# LLaMA-3-8B linear shapes (hidden 4096, intermediate 14336, 32/8 heads x 128):
# (site, K, N) for the four activation sites of one decoder layer.
LLAMA3_8B_SITES = [
    ("qkv", 4096, 6144),
    ("o", 4096, 4096),
    ("gate_up", 4096, 28672),
    ("down", 14336, 4096),
]

# LLaMA-3-70B (hidden 8192, intermediate 28672, 64/8 heads x 128), BASELINE configs[3]
LLAMA3_70B_SITES = [
    ("qkv", 8192, 10240),
    ("o", 8192, 8192),
    ("gate_up", 8192, 57344),
    ("down", 28672, 8192),
]
