"""Pins for the seeded input generators (readings C11, C14, C15, C16)."""
import json
import os

import numpy as np
import pytest

import sdnn_synth as synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def check_csr(p):
    rp, ci = p.row_ptr, p.col_idx
    assert rp.dtype == np.int32 and ci.dtype == np.int32 and p.vals.dtype == np.float32
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == ci.size == p.vals.size
    for m in range(p.M):
        seg = ci[rp[m]:rp[m + 1]]
        assert np.all(np.diff(seg) > 0)
    assert ci.size == 0 or (ci.min() >= 0 and ci.max() < p.K)
    assert not np.any(p.vals == 0)


@pytest.mark.parametrize("case", GOLD["generator"], ids=lambda c: c["cite"][:24])
def test_printed_nnz(case):
    assert synth.nnz_target(case["M"], case["K"], case["sparsity"]) == case["nnz"]
    p = synth.make_problem("g", case["M"], case["K"], 4, case["sparsity"])
    assert p.nnz == case["nnz"]
    check_csr(p)


EXPECTED_NNZ = {  # SURVEY.md §8(d) table (C11 / C15 integer rounding)
    "c1": 6554, "c2_768x768": 58982, "c2_3072x768": 235930, "c2_768x3072": 235930,
    "c3_128x64": 1229, "c3_256x128": 4915, "c3_512x512": 39322, "c3_1024x512": 78643,
    "c4_2048x512_s80": 209716, "c4_512x2048_s80": 209716, "c4_2048x512_s95": 52428,
    "c4_512x2048_s95": 52428, "c5": 1677722,
}


@pytest.mark.parametrize("key", [k for k in synth.CONFIGS if k != "c5"])
def test_config_nnz_and_validity(key):
    p = synth.config_problem(key, N=8)
    assert p.nnz == EXPECTED_NNZ[key]
    check_csr(p)
    if p.mask == "block4":
        # every nonzero belongs to an aligned 1x4 run (C15)
        d = p.dense_w() != 0
        blocks = d.reshape(p.M, p.K // 4, 4)
        assert np.all(blocks.all(-1) == blocks.any(-1))
    if p.mask == "lognormal":
        cnt = np.diff(p.row_ptr)
        assert cnt.max() <= p.K and cnt.max() > 4 * cnt.mean() / 2  # skewed (σ = 1)


@pytest.mark.slow
def test_c5_nnz():
    p = synth.config_problem("c5", N=8)
    assert p.nnz == EXPECTED_NNZ["c5"]


def test_determinism_and_seed_sensitivity():
    a = synth.config_problem("c1")
    b = synth.config_problem("c1")
    c = synth.config_problem("c1", seed=1)
    for f in ("row_ptr", "col_idx", "vals", "bias"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    np.testing.assert_array_equal(a.x(), b.x())
    assert not np.array_equal(a.col_idx, c.col_idx)


def test_x_shard_invariance():
    p = synth.make_problem("xs", 5, 7, 3 * synth.X_BLOCK + 123, 0.5)
    X = p.x()
    for c0, c1 in [(0, 10), (synth.X_BLOCK - 5, synth.X_BLOCK + 5), (100, 2 * synth.X_BLOCK + 7),
                   (3 * synth.X_BLOCK, p.N)]:
        np.testing.assert_array_equal(p.x_cols(c0, c1), X[:, c0:c1])


def test_lognormal_counts_exact_and_capped():
    rng = np.random.default_rng(0)
    c = synth.lognormal_row_counts(50, 10, 400, rng, sigma=2.0)
    assert c.sum() == 400 and c.max() <= 10


def test_value_distributions():
    p = synth.config_problem("c3_1024x512", N=64)
    assert abs(p.vals.std() - 0.05) < 0.002
    assert abs(p.bias.std() - 0.1) < 0.01
    X = p.x()
    assert abs(X.std() - 1.0) < 0.01 and abs(X.mean()) < 0.01


def test_threshold_mask_keeps_largest():
    p = synth.make_problem("thr", 40, 50, 2, 0.9, mask="threshold", seed=3)
    check_csr(p)
    assert p.nnz == synth.nnz_target(40, 50, 0.9)
    assert np.abs(p.vals).min() > 1.0  # 90 % quantile of |N(0,1)| ≈ 1.645
