"""The multi-GPU partition (BASELINE configs[4]) rehearsed on one GPU: c5's W with the
bench's full N = 262 144, and the column shards a rank owns at g = 2, 4 and 8 (contiguous K × N/g
tensors, bench.shard_range) run one after another through the same handle.  Y[:, n] depends only on
X[:, n] and every kernel sums each column in the same per-row order, so every shard's Y must equal the
unsharded Y on its columns bitwise — the property that makes the N-sharded job
collective-free.  Per-shard times are printed as a single-GPU proxy of per-rank efficiency."""
import os
import sys

import pytest
import torch

import sdnn_synth as synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


@pytest.fixture(scope="module")
def c5(sdnn):
    p = synth.config_problem("c5")
    h = sdnn.Handle.from_problem(p)
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn((p.K, p.N), device="cuda", generator=g)
    b = torch.from_numpy(p.bias).cuda()
    Y = h.spmm(X, b, act=1)
    torch.cuda.synchronize()
    yield p, h, X, b, Y
    h.close()


@pytest.mark.parametrize("g", [2, 4, 8])
def test_c5_shard_geometry_bitwise(c5, g):
    from bench import shard_range
    p, h, X, b, Y = c5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for r in range(g):
        c0, c1 = shard_range(p.N, r, g)
        assert c1 - c0 == p.N // g  # 4-aligned equal shards at the bench size
        Xs = X[:, c0:c1].contiguous()
        assert h.kernel_for(c1 - c0, Xs.data_ptr()) == h.kernel_for(p.N, X.data_ptr())  # the bench kernel
        Ys = h.spmm(Xs, b, act=1)
        e0.record()
        h.spmm(Xs, b, act=1, out=Ys)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        assert torch.equal(Ys, Y[:, c0:c1]), (g, r)
    print(f"c5 g={g}: per-shard ms (single-GPU proxy) {[round(t, 3) for t in times]}")
