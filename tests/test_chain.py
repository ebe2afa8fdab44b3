"""Cross-layer permutation: host-side pieces, no GPU.

* sdnn_csr_permute_columns gives the CSR of W·P — pinned against the dense matrix with its
  columns gathered by numpy (W·P)[:, i] = W[:, order[i]], not against itself;
* SDNN_FLAG_PERMUTED_OUTPUT maps every output slot of the plan to its position in the plan's
  Algorithm 1 order (row order[pos] = original row), and nothing else in the plan changes."""
import numpy as np
import pytest

import paper_2101_07948_b200 as sdnn
import sdnn_synth as synth


def dense(rp, ci, v, M, K):
    W = np.zeros((M, K), np.float64)
    for r in range(M):
        W[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    return W


@pytest.mark.parametrize("M,K,sp", [(40, 64, 0.7), (300, 200, 0.9), (1, 5, 0.0)])
def test_permute_columns_is_w_times_p(M, K, sp):
    p = synth.make_problem(f"pc{M}", M, K, 8, sp)
    order = np.random.default_rng(M).permutation(K).astype(np.int32)
    ci2, v2 = sdnn.permute_columns(p.row_ptr, p.col_idx, p.vals, M, K, order)
    W, W2 = dense(p.row_ptr, p.col_idx, p.vals, M, K), dense(p.row_ptr, ci2, v2, M, K)
    np.testing.assert_array_equal(W2, W[:, order])
    for r in range(M):  # rows stay strictly ascending (valid CSR)
        assert np.all(np.diff(ci2[p.row_ptr[r]:p.row_ptr[r + 1]]) > 0)


def test_permute_columns_identity_and_errors():
    p = synth.make_problem("pci", 50, 30, 8, 0.8)
    ci2, v2 = sdnn.permute_columns(p.row_ptr, p.col_idx, p.vals, 50, 30, np.arange(30))
    np.testing.assert_array_equal(ci2, p.col_idx)
    np.testing.assert_array_equal(v2, p.vals)
    bad = np.arange(30)
    bad[3] = 4  # not a bijection
    with pytest.raises(sdnn.SdnnError):
        sdnn.permute_columns(p.row_ptr, p.col_idx, p.vals, 50, 30, bad)
    with pytest.raises(ValueError):
        sdnn.permute_columns(p.row_ptr, p.col_idx, p.vals, 50, 30, np.arange(29))


@pytest.mark.parametrize("kernel", ["row", "tmem", "tmem8", "group"])
@pytest.mark.parametrize("key", ["c2_768x768", "c3_512x512"])
def test_permuted_output_maps_slots_to_positions(key, kernel):
    p = synth.config_problem(key)
    a = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel=kernel)
    b = sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel=kernel, permuted_output=True)
    order = sdnn.permutation(p.row_ptr, p.col_idx, p.M, p.K)
    pos = np.empty(p.M, np.int64)
    pos[order] = np.arange(p.M)
    ra, oa, ma = a.export()
    rb, ob, mb = b.export()
    np.testing.assert_array_equal(oa, ob)  # the execution-ordered stream is unchanged
    np.testing.assert_array_equal(ma, mb)
    np.testing.assert_array_equal(rb[ra >= 0], pos[ra[ra >= 0]])
    np.testing.assert_array_equal(rb[ra < 0], ra[ra < 0])  # empty slots / pieces keep their codes


def test_permuted_output_not_with_codegen():
    p = synth.config_problem("c1")
    with pytest.raises(sdnn.SdnnError) as e:
        sdnn.Plan(p.row_ptr, p.col_idx, p.vals, p.M, p.K, kernel="codegen", permuted_output=True)
    assert e.value.status == 3
