"""Chained layers with the permutation carried across layers,
through the C ABI on the GPU.

* A layer prepared with SDNN_FLAG_PERMUTED_OUTPUT writes Y[order] (bias given in plan order) —
  bitwise the permuted rows of the ordinary call (same per-row accumulation order);
* a chain (every layer but the last with permuted output, next layer's columns relabelled) equals
  the layer-by-layer result: the last layer is checked against the oracle applied to the GPU's own
  intermediate (bitwise the un-chained intermediate, permuted), with the north_star tolerance."""
import numpy as np
import pytest

import sdnn_synth as synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


def parity(Y, Yo, S):
    zero = S == 0
    assert np.all(Y[zero] == Yo[zero])
    err = np.abs(Y.astype(np.float64) - Yo) / np.where(zero, 1.0, S)
    assert float(err.max()) <= TOL, float(err.max())


@pytest.mark.parametrize("kernel", ["auto", "row", "tmem", "group"])
@pytest.mark.parametrize("key,N", [("c2_768x768", 1024), ("c2_768x768", 100), ("c3_512x512", 512),
                                   ("c2_768x3072", 1024)])  # the last: TMEM split-K under auto
def test_permuted_output_is_permuted_rows(sdnn, key, N, kernel):
    p = synth.config_problem(key)
    X = torch.from_numpy(np.ascontiguousarray(p.x()[:, :N])).cuda()
    b = torch.from_numpy(p.bias).cuda()
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    hp = sdnn.Handle.from_problem(p, kernel=kernel, permuted_output=True)
    order = hp.permutation()
    np.testing.assert_array_equal(order, h.permutation())
    Y = h.spmm(X, b, act=1).cpu().numpy()
    bp = torch.from_numpy(np.ascontiguousarray(p.bias[order])).cuda()
    Yp = hp.spmm(X, bp, act=1).cpu().numpy()
    np.testing.assert_array_equal(Yp, Y[order])


@pytest.mark.parametrize("N", [1024, 200])
def test_ffn_chain(sdnn, oracle_mod, N):
    """BERT FFN pair at c2's shapes (768 → 3072 → 768, 90 %, log-normal rows), ReLU between."""
    w1 = synth.config_problem("c2_3072x768")  # M = 3072, K = 768
    w2 = synth.config_problem("c2_768x3072")  # M = 768,  K = 3072
    chain = sdnn.Chain([(w1.row_ptr, w1.col_idx, w1.vals, w1.M, w1.K, w1.bias, 1),
                        (w2.row_ptr, w2.col_idx, w2.vals, w2.M, w2.K, w2.bias, 1)])
    X = torch.from_numpy(np.ascontiguousarray(w1.x()[:, :N])).cuda()
    Yc = chain.forward(X).cpu().numpy()
    h1, h2 = sdnn.Handle.from_problem(w1), sdnn.Handle.from_problem(w2)
    Y1 = h1.spmm(X, torch.from_numpy(w1.bias).cuda(), act=1)
    # the chain's intermediate is bitwise the un-chained one in layer 1's plan order
    np.testing.assert_array_equal(chain._bufs[N][0].cpu().numpy(), Y1.cpu().numpy()[chain.handles[0].permutation()])
    Y1h = Y1.cpu().numpy()
    Yo, S = oracle_mod.spmm_omp(w2.row_ptr, w2.col_idx, w2.vals, w2.M, w2.K, Y1h, w2.bias, act=1, want_scale=True)[:2]
    parity(Yc, Yo, S)
    Yu = h2.spmm(Y1, torch.from_numpy(w2.bias).cuda(), act=1).cpu().numpy()
    parity(Yu, Yo, S)


def test_three_layer_chain_no_act(sdnn, oracle_mod):
    ps = [synth.make_problem("ch0", 256, 128, 64, 0.8), synth.make_problem("ch1", 192, 256, 64, 0.9),
          synth.make_problem("ch2", 100, 192, 64, 0.85)]
    chain = sdnn.Chain([(q.row_ptr, q.col_idx, q.vals, q.M, q.K, None if i == 1 else q.bias, 0)
                        for i, q in enumerate(ps)], kernel="row")
    X = ps[0].x()
    Yc = chain.forward(torch.from_numpy(X).cuda()).cpu().numpy()
    # layer by layer on the GPU (un-chained), then the oracle on the last intermediate
    cur = torch.from_numpy(X).cuda()
    for i, q in enumerate(ps[:-1]):
        b = None if i == 1 else torch.from_numpy(q.bias).cuda()
        cur = sdnn.Handle.from_problem(q, kernel="row").spmm(cur, b, act=0)
    q = ps[-1]
    Yo, S = oracle_mod.spmm_omp(q.row_ptr, q.col_idx, q.vals, q.M, q.K, cur.cpu().numpy(), q.bias, act=0,
                                want_scale=True)[:2]
    parity(Yc, Yo, S)
    with pytest.raises(ValueError):
        sdnn.Chain([(ps[0].row_ptr, ps[0].col_idx, ps[0].vals, ps[0].M, ps[0].K, None, 0),
                    (ps[2].row_ptr, ps[2].col_idx, ps[2].vals, ps[2].M, ps[2].K, None, 0)])
