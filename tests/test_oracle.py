"""Pins for the CPU oracle.  Nothing here compares the oracle with itself:
every expected value is a printed worked example (tests/golden, cited), a closed form, a brute
force, or a library routine (numpy dense fp64 matmul, scipy.sparse)."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
from hypothesis import given, settings, strategies as st

import sdnn_synth as synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def csr_of(dense):
    d = np.asarray(dense, dtype=np.float32)
    m = sp.csr_matrix(d)
    m.sort_indices()
    return m.indptr.astype(np.int32), m.indices.astype(np.int32), m.data.astype(np.float32)


def csr_keep_pattern(dense_vals, mask):
    """CSR with an explicit pattern (allows stored zeros)."""
    M, K = mask.shape
    rp = np.zeros(M + 1, np.int32)
    rp[1:] = np.cumsum(mask.sum(1))
    r, c = np.nonzero(mask)
    return rp, c.astype(np.int32), dense_vals[r, c].astype(np.float32)


def library_ref(W, X, b, act):
    """numpy fp64 dense product + bias + act, rounded once to fp32 (P3 library routine)."""
    v = W.astype(np.float64) @ X.astype(np.float64)
    if b is not None:
        v = v + b.astype(np.float64)[:, None]
    if act == 1:
        v = np.where(v > 0, v, 0.0)
    S = np.abs(W.astype(np.float64)) @ np.abs(X.astype(np.float64))
    if b is not None:
        S = S + np.abs(b.astype(np.float64))[:, None]
    return v.astype(np.float32), S


def assert_within_fp64_rounding(Y, Yref, S):
    """Both are fp64 sums rounded once to fp32; only summation order differs → ≤ 1 ulp, or a tiny
    absolute slack near zero (K·2^-53·S)."""
    tol = np.maximum(np.spacing(np.abs(Yref).astype(np.float32)).astype(np.float64), 1e-12 * S)
    assert np.all(np.abs(Y.astype(np.float64) - Yref.astype(np.float64)) <= tol)


# ---------------------------------------------------------------- P1: printed worked values
@pytest.mark.parametrize("case", GOLD["spmm"], ids=lambda c: c["cite"][:24])
def test_worked_examples(oracle_mod, case):
    W = np.array(case["W"], np.float32)
    X = np.array(case["X"], np.float32)
    rp, ci, v = csr_of(W)
    Y, S = oracle_mod.spmm(rp, ci, v, W.shape[0], W.shape[1], X, None, act=0)
    np.testing.assert_array_equal(Y, np.array(case["Y"], np.float32))


@pytest.mark.parametrize("case", GOLD["csr"], ids=lambda c: c["cite"][:24])
def test_csr_fixtures(case):
    rp, ci, v = csr_of(case["W"])
    assert rp.tolist() == case["row_ptr"] and ci.tolist() == case["col_idx"] and v.tolist() == case["vals"]


# ---------------------------------------------------------------- P2: closed forms
@pytest.mark.parametrize("N", [1, 2, 3, 5, 17])
def test_identity_closed_form(oracle_mod, N):
    rng = np.random.default_rng(1)
    M = 7
    X = rng.standard_normal((M, N)).astype(np.float32)
    b = rng.standard_normal(M).astype(np.float32)
    rp, ci, v = csr_of(np.eye(M))
    for act in (0, 1):
        Y, S = oracle_mod.spmm(rp, ci, v, M, M, X, b, act=act)
        ref = (X.astype(np.float64) + b[:, None]).astype(np.float64)
        if act:
            ref = np.maximum(ref, 0)
        np.testing.assert_array_equal(Y, ref.astype(np.float32))  # one product, one add: exact fp64
        np.testing.assert_array_equal(S, np.abs(X.astype(np.float64)) + np.abs(b.astype(np.float64))[:, None])


def test_empty_w_gives_act_bias(oracle_mod):
    M, K, N = 5, 9, 4
    rp = np.zeros(M + 1, np.int32)
    b = np.array([-1.5, 0.0, 2.25, -0.0, 3.0], np.float32)
    X = np.ones((K, N), np.float32)
    Y, S = oracle_mod.spmm(rp, np.zeros(0, np.int32), np.zeros(0, np.float32), M, K, X, b, act=1)
    np.testing.assert_array_equal(Y, np.repeat(np.maximum(b, 0)[:, None], N, 1))
    np.testing.assert_array_equal(S, np.repeat(np.abs(b.astype(np.float64))[:, None], N, 1))
    Y0, S0 = oracle_mod.spmm(rp, np.zeros(0, np.int32), np.zeros(0, np.float32), M, K, X, None, act=0)
    assert not Y0.any() and not S0.any()


def test_single_nonzero(oracle_mod):
    M, K, N = 6, 11, 9
    rng = np.random.default_rng(2)
    X = rng.standard_normal((K, N)).astype(np.float32)
    b = rng.standard_normal(M).astype(np.float32)
    W = np.zeros((M, K), np.float32)
    W[3, 7] = -0.625  # exactly representable: w·x exact in fp32 too
    rp, ci, v = csr_of(W)
    Y, _ = oracle_mod.spmm(rp, ci, v, M, K, X, b, act=1)
    for m in range(M):
        ref = (np.float64(-0.625) * X[7].astype(np.float64) if m == 3 else 0.0) + np.float64(b[m])
        np.testing.assert_array_equal(Y[m], np.maximum(ref, 0).astype(np.float32))


def test_all_ones_x_gives_row_sums(oracle_mod):
    p = synth.make_problem("ones", 40, 33, 6, 0.7, seed=3)
    X = np.ones((p.K, p.N), np.float32)
    Y, _ = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    rows = np.array([math_fsum(p.vals[p.row_ptr[m]:p.row_ptr[m + 1]]) for m in range(p.M)])
    ref = np.maximum(rows + p.bias.astype(np.float64), 0).astype(np.float32)
    Yref = np.repeat(ref[:, None], p.N, 1)
    S = np.abs(p.dense_w()).astype(np.float64).sum(1)[:, None] + np.abs(p.bias)[:, None]
    assert_within_fp64_rounding(Y, Yref, np.repeat(S, p.N, 1))


def math_fsum(a):
    import math
    return math.fsum(float(x) for x in a)


def test_linearity_power_of_two_exact(oracle_mod):
    """act = NONE, bias = NULL: Y(2X) = 2·Y(X) bitwise (scaling by 2 is exact in fp64 and fp32)."""
    p = synth.make_problem("lin", 50, 70, 13, 0.8, seed=4)
    X = p.x()
    Y1, S1 = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, None, act=0)
    Y2, S2 = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, 2 * X, None, act=0)
    np.testing.assert_array_equal(Y2, 2 * Y1)
    np.testing.assert_array_equal(S2, 2 * S1)


def test_relu_and_none_agree_on_positive(oracle_mod):
    p = synth.make_problem("relu", 30, 30, 8, 0.5, seed=5)
    X = p.x()
    Yn, _ = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=0)
    Yr, _ = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    np.testing.assert_array_equal(Yr, np.where(Yn > 0, Yn, 0).astype(np.float32))
    assert (Yn < 0).any() and (Yn > 0).any()


# ---------------------------------------------------------------- P3: dense extreme vs library
@pytest.mark.parametrize("shape", [(16, 24, 5), (64, 48, 33), (3, 200, 7)])
def test_dense_matches_numpy(oracle_mod, shape):
    M, K, N = shape
    rng = np.random.default_rng(M * K)
    W = (0.05 * rng.standard_normal((M, K))).astype(np.float32)
    W[W == 0] = 0.01
    X = rng.standard_normal((K, N)).astype(np.float32)
    b = (0.1 * rng.standard_normal(M)).astype(np.float32)
    rp, ci, v = csr_of(W)
    assert rp[-1] == M * K
    for act in (0, 1):
        Y, S = oracle_mod.spmm(rp, ci, v, M, K, X, b, act=act)
        Yref, Sref = library_ref(W, X, b, act)
        assert_within_fp64_rounding(Y, Yref, Sref)
        np.testing.assert_allclose(S, Sref, rtol=1e-12, atol=0)


def test_transposed_operand_would_fail(oracle_mod):
    """Guard that P3's comparison is sensitive: a rectangular W with the wrong orientation differs."""
    rng = np.random.default_rng(9)
    W = rng.standard_normal((5, 8)).astype(np.float32)
    X = rng.standard_normal((8, 3)).astype(np.float32)
    rp, ci, v = csr_of(W)
    Y, S = oracle_mod.spmm(rp, ci, v, 5, 8, X, None, act=0)
    Yref, Sref = library_ref(W, X, None, 0)
    assert_within_fp64_rounding(Y, Yref, Sref)
    Wbad = W.copy(); Wbad[0, 0] = -Wbad[0, 0]
    Ybad, _ = library_ref(Wbad, X, None, 0)
    assert np.abs(Y - Ybad).max() > 1e-3


# ---------------------------------------------------------------- P4: random tiny vs scipy
@settings(max_examples=150, deadline=None)
@given(M=st.integers(1, 24), K=st.integers(1, 24), N=st.integers(1, 12),
       dens=st.floats(0.0, 1.0), seed=st.integers(0, 2**31 - 1), act=st.integers(0, 1),
       with_bias=st.booleans())
def test_random_tiny_vs_scipy(oracle_mod, M, K, N, dens, seed, act, with_bias):
    rng = np.random.default_rng(seed)
    mask = rng.random((M, K)) < dens
    vals = (0.05 * rng.standard_normal((M, K))).astype(np.float32)
    rp, ci, v = csr_keep_pattern(vals, mask)  # stored zeros allowed (reading C6)
    X = rng.standard_normal((K, N)).astype(np.float32)
    b = (0.1 * rng.standard_normal(M)).astype(np.float32) if with_bias else None
    Y, S = oracle_mod.spmm(rp, ci, v, M, K, X, b, act=act)
    Wsp = sp.csr_matrix((v.astype(np.float64), ci, rp), shape=(M, K))
    ref = np.asarray(Wsp @ X.astype(np.float64))
    if b is not None:
        ref = ref + b.astype(np.float64)[:, None]
    if act:
        ref = np.where(ref > 0, ref, 0.0)
    Sref = np.asarray(abs(Wsp) @ np.abs(X.astype(np.float64)))
    if b is not None:
        Sref = Sref + np.abs(b.astype(np.float64))[:, None]
    assert_within_fp64_rounding(Y, ref.astype(np.float32), Sref)
    np.testing.assert_allclose(S, Sref, rtol=1e-12, atol=1e-300)


# ---------------------------------------------------------------- P5: permutation invariance
def test_row_permutation_roundtrip_bitwise(oracle_mod):
    p = synth.make_problem("perm", 64, 80, 19, 0.9, mask="lognormal", seed=6)
    X = p.x()
    Y, S = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    perm = np.random.default_rng(7).permutation(p.M)
    counts = np.diff(p.row_ptr)[perm]
    rp = np.zeros(p.M + 1, np.int32); rp[1:] = np.cumsum(counts)
    ci = np.concatenate([p.col_idx[p.row_ptr[r]:p.row_ptr[r + 1]] for r in perm])
    v = np.concatenate([p.vals[p.row_ptr[r]:p.row_ptr[r + 1]] for r in perm])
    Yp, Sp = oracle_mod.spmm(rp, ci, v, p.M, p.K, X, p.bias[perm], act=1)
    Yun = np.empty_like(Yp); Yun[perm] = Yp
    Sun = np.empty_like(Sp); Sun[perm] = Sp
    np.testing.assert_array_equal(Yun, Y)
    np.testing.assert_array_equal(Sun, S)


def test_column_independence_bitwise(oracle_mod):
    p = synth.make_problem("cols", 33, 45, 40, 0.85, seed=8)
    X = p.x()
    Y, _ = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    Ya, _ = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X[:, :13], p.bias, act=1)
    Yb, _ = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X[:, 13:], p.bias, act=1)
    np.testing.assert_array_equal(np.concatenate([Ya, Yb], 1), Y)


def test_omp_variant_bitwise(oracle_mod):
    p = synth.make_problem("omp", 300, 200, 37, 0.9, mask="lognormal", seed=9)
    X = p.x()
    Y, S = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    Yo, So, used = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1, threads=4,
                                       want_scale=True)
    assert used >= 1
    np.testing.assert_array_equal(Yo, Y)
    np.testing.assert_array_equal(So, S)


def test_bad_act_rejected(oracle_mod):
    rp, ci, v = csr_of(np.eye(2))
    with pytest.raises(RuntimeError):
        oracle_mod.spmm(rp, ci, v, 2, 2, np.ones((2, 2), np.float32), None, act=7)


# ---------------------------------------------------------------- P6: Algorithm 1
@pytest.mark.parametrize("case", GOLD["alg1"], ids=lambda c: c["cite"][:24])
def test_alg1_printed_traces(oracle_mod, case):
    rows = [set(r) for r in case["rows"]]
    assert oracle_mod.alg1_bruteforce(rows) == case["order"]
    K = case["K"]
    W = np.zeros((len(rows), K), np.float32)
    for i, r in enumerate(rows):
        W[i, list(r)] = 1
    rp, ci, _ = csr_of(W)
    assert oracle_mod.alg1(rp, ci, len(rows), K).tolist() == case["order"]


def _check_greedy_property(order, dense_mask):
    """Independent check of each step of Algorithm 1 from the dense mask: position 0 has maximal nnz
    (lowest index among ties) and each next row has maximal overlap with its predecessor among the
    rows not yet placed (lowest index among ties)."""
    M = dense_mask.shape[0]
    assert sorted(order) == list(range(M))  # bijection
    nnz = dense_mask.sum(1)
    assert order[0] == int(np.flatnonzero(nnz == nnz.max())[0])
    placed = np.zeros(M, bool); placed[order[0]] = True
    for i in range(1, M):
        ov = (dense_mask & dense_mask[order[i - 1]]).sum(1).astype(np.int64)
        ov[placed] = -1
        assert order[i] == int(np.flatnonzero(ov == ov.max())[0])
        placed[order[i]] = True


@pytest.mark.parametrize("seed", range(200))
def test_alg1_c_matches_bruteforce(oracle_mod, seed):
    rng = np.random.default_rng(1000 + seed)
    M = int(rng.integers(1, 30)); K = int(rng.integers(1, 30))
    mask = rng.random((M, K)) < rng.uniform(0.0, 0.6)
    if seed % 7 == 0:  # force duplicated rows and empty rows (tie handling)
        mask[M // 2:] = mask[: M - M // 2]
        mask[0] = False
    rp, ci, _ = csr_keep_pattern(np.ones((M, K), np.float32), mask)
    order_c = oracle_mod.alg1(rp, ci, M, K).tolist()
    order_py = oracle_mod.alg1_bruteforce([set(np.flatnonzero(mask[i]).tolist()) for i in range(M)])
    assert order_c == order_py
    _check_greedy_property(order_c, mask)


def test_alg1_lognormal_property(oracle_mod):
    p = synth.make_problem("alg1ln", 200, 150, 1, 0.9, mask="lognormal", seed=11)
    order = oracle_mod.alg1(p.row_ptr, p.col_idx, p.M, p.K).tolist()
    _check_greedy_property(order, p.dense_w() != 0)
