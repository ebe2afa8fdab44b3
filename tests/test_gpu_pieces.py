"""Heavy rows split into pieces on the warps of one CTA (reading R4): the row kernel adds a
row's pieces in shared memory at its end; on the generic path (ragged N) the pieces go through the
workspace and split_reduce_kernel.  Oracle parity (|Y − Y_oracle| ≤ 1e-4·S) and run-to-run bitwise
determinism on matrices built to stress it: rows with K and K/2 nonzeros among 1 % rows, twelve
K-dense rows, N tiles of 64 / 128 / 256 columns and a ragged N, K chunks of 64 and 8 (the stage ring
that holds the pieces' sums is then 8 K rows deep)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


def csr_from_mask(mask, rng):
    rows, cols = np.nonzero(mask)
    rp = np.zeros(mask.shape[0] + 1, np.int32)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    vals = (0.05 * rng.standard_normal(cols.size)).astype(np.float32)
    vals[vals == 0] = 0.01
    return rp, cols.astype(np.int32), vals


def heavy_one(rng):
    M, K = 96, 4096
    mask = rng.random((M, K)) < 0.01
    mask[5, :] = True            # one row with K nonzeros
    mask[50, ::2] = True         # one half-dense row
    return M, K, mask


def heavy_many(rng):
    M, K = 512, 4096
    mask = rng.random((M, K)) < 0.01
    mask[rng.choice(M, 12, replace=False)] = True  # twelve rows with K nonzeros (4 pieces each)
    return M, K, mask


@pytest.mark.parametrize("shape", ["one", "many"])
@pytest.mark.parametrize("N", [64, 1024, 2050, 8192])
@pytest.mark.parametrize("k_chunk", [0, 8])
def test_split_rows_parity(sdnn, oracle_mod, shape, N, k_chunk):
    rng = np.random.default_rng(7)
    M, K, mask = heavy_one(rng) if shape == "one" else heavy_many(rng)
    rp, ci, v = csr_from_mask(mask, rng)
    X = rng.standard_normal((K, N)).astype(np.float32)
    b = (0.1 * rng.standard_normal(M)).astype(np.float32)
    h = sdnn.Handle(rp, ci, v, M, K, kernel="row", k_chunk=k_chunk)
    assert h.info()["num_split_rows"] > 0
    Y = h.spmm(torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda(), act=1).cpu().numpy()
    Y2 = h.spmm(torch.from_numpy(X).cuda(), torch.from_numpy(b).cuda(), act=1).cpu().numpy()
    np.testing.assert_array_equal(Y, Y2)  # deterministic piece order
    Yo, S = oracle_mod.spmm_omp(rp, ci, v, M, K, X, b, act=1, want_scale=True)[:2]
    zero = S == 0
    assert np.all(Y[zero] == Yo[zero])
    err = np.abs(Y.astype(np.float64) - Yo) / np.where(zero, 1.0, S)
    assert float(err.max()) <= TOL, float(err.max())
