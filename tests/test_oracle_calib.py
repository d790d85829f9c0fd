"""Pins for the oracle's calibration ("Adaptive Outlier Identification", P:584 tau = 2^-3 M)."""
import json
import os

import numpy as np
import torch

import oracle
from paper_2601_07475_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_example_tau_rule():
    g = json.load(open(os.path.join(GOLDEN, "calibration_spec_example.json")))
    p = oracle.select_outliers(np.array(g["chan_max"], np.float32))
    assert p["M"] == g["M"] and p["tau"] == g["tau"]
    assert p["S_raw"] == g["S_raw"] and p["S"] == g["S"]
    assert list(p["perm"][:4]) == g["perm_prefix"]
    assert sorted(p["perm"]) == list(range(16))


def test_all_equal_and_all_zero():
    # every channel equal -> all strictly above tau = M/8; all zero -> S = 0
    p = oracle.select_outliers(np.full(64, 3.0, np.float32))
    assert p["S_raw"] == 64 and p["S"] == 64 and list(p["perm"]) == list(range(64))
    p = oracle.select_outliers(np.zeros(64, np.float32))
    assert p["S_raw"] == 0 and p["S"] == 0 and p["M"] == 0 and p["gs"] == 1.0


def test_perm_prefix_is_the_selected_set_and_sorted():
    rng = np.random.default_rng(0)
    for _ in range(50):
        K = int(rng.integers(1, 40)) * 16
        cm = (np.exp(rng.uniform(-4, 3, K)) * (rng.random(K) < 0.9)).astype(np.float32)
        cm[rng.integers(0, K, 3)] = cm[rng.integers(0, K)]  # ties
        p = oracle.select_outliers(cm)
        perm, sr, tau = p["perm"], p["S_raw"], p["tau"]
        assert sorted(perm) == list(range(K))
        assert set(perm[:sr].tolist()) == set(np.nonzero(cm > tau)[0].tolist())
        v = cm[perm]
        assert np.all(v[:-1] >= v[1:])                                        # descending
        ties = (v[:-1] == v[1:])
        assert np.all(perm[:-1][ties] < perm[1:][ties])                        # ties -> lower index
        assert p["S"] == min(K, (sr + 15) // 16 * 16)
        assert p["tau"] == np.float32(p["M"]) * np.float32(0.125)
        assert p["gs"] == (np.float32(2688.0) / np.float32(p["M"]) if p["M"] > 0 else 1.0)


def test_override_and_errors():
    cm = np.exp(np.random.default_rng(1).uniform(-2, 2, 128)).astype(np.float32)
    assert oracle.select_outliers(cm, 32)["S"] == 32
    for bad in (17, 144):
        try:
            oracle.select_outliers(cm, bad)
            raise AssertionError("expected shape error")
        except oracle.OracleError:
            pass
    cm[3] = np.nan
    try:
        oracle.select_outliers(cm)
        raise AssertionError("expected non-finite error")
    except oracle.OracleError:
        pass


def test_absmax_is_exact_column_max():
    x = synth.activation(300, 128, synth.Structure(128, 4, 0), seed=3)
    cm = oracle.calib_absmax(oracle.as_bf16_bits(x))
    assert np.array_equal(cm, x.float().abs().amax(0).numpy())
    # max aggregation across batches
    cm2 = oracle.calib_absmax(oracle.as_bf16_bits(x[150:]), oracle.calib_absmax(oracle.as_bf16_bits(x[:150])))
    assert np.array_equal(cm, cm2)


def test_synthetic_structure_recovered():
    """With >= 32x outlier gains the tau rule selects exactly the injected channels
    (DESIGN.md input recipe)."""
    K, S_inj = 1024, 32
    st = synth.Structure(K, S_inj, seed=0)
    cal = synth.activation(2048, K, st, seed=1000)
    p = oracle.select_outliers(oracle.calib_absmax(oracle.as_bf16_bits(cal)))
    assert p["S_raw"] == S_inj and p["S"] == S_inj
    assert set(p["perm"][:S_inj].tolist()) == set(st.idx.tolist())
