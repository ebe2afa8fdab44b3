"""GPU parity: libsdnn (through the C ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star; reading C9): |Y_gpu − Y_oracle| ≤ 1e-4 · S per element,
S = Σ|w||x| + |b| from the oracle; exact equality where S = 0.  Invariants that hold bitwise (fixed
per-row accumulation order) are checked bitwise."""
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


def run_gpu(sdnn, p, X, bias=None, act=1, handle=None, **opts):
    h = handle or sdnn.Handle.from_problem(p, **opts)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    bd = None if bias is None else torch.from_numpy(bias).cuda()
    Y = h.spmm(Xd, bd, act=act)
    torch.cuda.synchronize()
    return Y.cpu().numpy(), h


def assert_parity(Y, Yo, S, what=""):
    err = np.abs(Y.astype(np.float64) - Yo.astype(np.float64))
    zero = S == 0
    assert np.all(Y[zero] == Yo[zero]), f"{what}: nonzero output where S = 0"
    ratio = np.where(zero, 0.0, err / np.where(zero, 1.0, S))
    worst = float(ratio.max()) if ratio.size else 0.0
    assert worst <= TOL, f"{what}: max |err|/S = {worst:.3e} > {TOL}"
    return worst


def check(sdnn, oracle_mod, p, X=None, act=None, bias="p", **opts):
    X = p.x() if X is None else X
    b = p.bias if isinstance(bias, str) else bias
    act = p.act if act is None else act
    Y, h = run_gpu(sdnn, p, X, b, act, **opts)
    Yo, S = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, b, act=act, want_scale=True)[:2]
    return assert_parity(Y, Yo, S, p.name), Y, h


# ------------------------------------------------------------------ worked examples (P1)
def test_worked_example(sdnn, oracle_mod):
    W = np.array([[0, 2], [3, 0]], np.float32)
    rp, ci, v = np.array([0, 1, 2], np.int32), np.array([1, 0], np.int32), np.array([2, 3], np.float32)
    h = sdnn.Handle(rp, ci, v, 2, 2)
    Y = h.spmm(torch.ones(2, 2, device="cuda"), None, act=0).cpu().numpy()
    np.testing.assert_array_equal(Y, [[2, 2], [3, 3]])


# ------------------------------------------------------------------ BASELINE configs c1-c4 (full size)
@pytest.mark.parametrize("kernel", ["auto", "row", "group1", "group2", "group4", "codegen", "tmem", "tmem8", "tmemp"])
@pytest.mark.parametrize("key", [k for k in synth.CONFIGS if k != "c5"])
def test_config_parity(sdnn, oracle_mod, key, kernel):
    p = synth.config_problem(key)
    kw = dict(kernel="group", group_sb=int(kernel[-1])) if kernel.startswith("group") else dict(kernel=kernel)
    worst, _, h = check(sdnn, oracle_mod, p, **kw)
    print(f"{key} {kernel}->{h.info()['kernel']}: max err/S = {worst:.2e}")


def test_c2_no_act(sdnn, oracle_mod):
    p = synth.config_problem("c2_3072x768", act=0)
    check(sdnn, oracle_mod, p)


# ------------------------------------------------------------------ desk grid
@pytest.mark.parametrize("kernel", ["row", "group", "codegen", "tmem", "tmem8", "tmemp"])
@pytest.mark.parametrize("g", list(synth.desk_grid()), ids=lambda g: f"{g['name']}_s{g['seed']}")
def test_desk_grid(sdnn, oracle_mod, g, kernel):
    p = synth.make_problem(g["name"], g["M"], g["K"], g["N"], g["sparsity"], seed=g["seed"])
    check(sdnn, oracle_mod, p, kernel=kernel)


# ------------------------------------------------------------------ c5 at full size, launch config of bench.py
@pytest.mark.parametrize("kernel", ["auto", "row", "codegen", "tmem", "tmem8", "tmemp"])
def test_c5_full_size_sampled_columns(sdnn, oracle_mod, kernel):
    p = synth.config_problem("c5")
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    X = torch.empty((p.K, p.N), dtype=torch.float32, device="cuda")
    for b in range((p.N + synth.X_BLOCK - 1) // synth.X_BLOCK):
        blk = torch.from_numpy(p.x_block(b))
        X[:, b * synth.X_BLOCK:b * synth.X_BLOCK + blk.shape[1]].copy_(blk)
    bias = torch.from_numpy(p.bias).cuda()
    Y = h.spmm(X, bias, act=1)
    cols = np.concatenate([np.arange(0, 64), np.arange(131072 - 32, 131072 + 32), np.arange(p.N - 64, p.N),
                           np.random.default_rng(0).choice(p.N, 64, replace=False)])
    cols_t = torch.from_numpy(cols).cuda()
    Ys = Y[:, cols_t].cpu().numpy()
    Xs = X[:, cols_t].cpu().numpy()
    Yo, S, _ = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, Xs, p.bias, act=1, want_scale=True)
    assert_parity(Ys, Yo, S, "c5 sampled")


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("kernel", ["row", "group", "codegen", "tmem", "tmem8", "tmemp"])
@pytest.mark.parametrize("N", [1, 2, 3, 5, 7, 13, 127, 128, 129, 256, 300, 384, 1000, 1024])
def test_ragged_n(sdnn, oracle_mod, N, kernel):
    p = synth.make_problem("ragged", 200, 150, N, 0.9, mask="lognormal", seed=N)
    check(sdnn, oracle_mod, p, kernel=kernel)


@pytest.mark.parametrize("kernel", ["tmem", "tmemp"])
@pytest.mark.parametrize("N", [4, 100, 132, 1000, 6276])
def test_tmem_fast_path_partial_tiles(sdnn, oracle_mod, N, kernel):
    """TMEM-R kernels (2-D tensor map) take any N % 4 == 0 on the fast path: the last 128-column
    tile's columns past N are zero-filled by TMA and not stored — oracle parity, and bitwise equal to
    the same columns of a call with N rounded up to whole tiles (column independence)."""
    p = synth.make_problem("ptile", 600, 700, N, 0.9, seed=N)
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    assert h.kernel_for(N, 256, 256) == (6 if kernel == "tmemp" else 4)
    check(sdnn, oracle_mod, p, kernel=kernel)
    Nr = (N + 127) // 128 * 128
    X = np.zeros((p.K, Nr), np.float32)
    X[:, :N] = p.x()
    Y, _ = run_gpu(sdnn, p, np.ascontiguousarray(X[:, :N]), p.bias, 1, handle=h)
    Yr, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    np.testing.assert_array_equal(Y, Yr[:, :N])


@pytest.mark.parametrize("kernel", ["row", "group", "codegen", "tmem", "tmem8", "tmemp"])
def test_unaligned_pointers(sdnn, oracle_mod, kernel):
    p = synth.make_problem("unal", 100, 90, 64, 0.8, seed=1)
    X = p.x()
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    Xbuf = torch.zeros(p.K * p.N + 1, device="cuda")
    Xbuf[1:].copy_(torch.from_numpy(X).reshape(-1))
    Ybuf = torch.zeros(p.M * p.N + 1, device="cuda")
    Xv = Xbuf[1:].view(p.K, p.N)
    Yv = Ybuf[1:].view(p.M, p.N)
    h.spmm(Xv, torch.from_numpy(p.bias).cuda(), act=1, out=Yv)
    Yo, S = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    assert_parity(Yv.cpu().numpy(), Yo, S, "unaligned")


@pytest.mark.parametrize("kernel", ["row", "group", "codegen", "tmem", "tmem8", "tmemp"])
@pytest.mark.parametrize("M,K,N,dens", [(1, 1, 4, 1.0), (1, 500, 8, 0.3), (500, 1, 8, 0.5), (37, 65, 12, 1.0),
                                        (129, 257, 20, 0.0), (64, 64, 64, 1.0), (2100, 70, 40, 0.05),
                                        (1, 500, 128, 0.3), (500, 1, 256, 0.5), (129, 257, 384, 0.0),
                                        (2100, 70, 128, 0.05), (65, 300, 1024, 1.0)])
def test_degenerate_shapes(sdnn, oracle_mod, M, K, N, dens, kernel):
    rng = np.random.default_rng(M + K + N)
    mask = rng.random((M, K)) < dens
    rp = np.zeros(M + 1, np.int32); rp[1:] = np.cumsum(mask.sum(1))
    ci = np.nonzero(mask)[1].astype(np.int32)
    v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
    b = (0.1 * rng.standard_normal(M)).astype(np.float32)
    p = synth.Problem("deg", M, K, N, 0, "x", rp, ci, v, b, 1, 0)
    X = rng.standard_normal((K, N)).astype(np.float32)
    for act in (0, 1):
        check(sdnn, oracle_mod, p, X=X, act=act, kernel=kernel)
    check(sdnn, oracle_mod, p, X=X, act=1, bias=None, kernel=kernel)


def test_empty_weight(sdnn, oracle_mod):
    M, K, N = 70, 40, 24
    p = synth.Problem("empty", M, K, N, 1.0, "x", np.zeros(M + 1, np.int32), np.zeros(0, np.int32),
                      np.zeros(0, np.float32), np.linspace(-1, 1, M).astype(np.float32), 1, 0)
    X = np.random.default_rng(0).standard_normal((K, N)).astype(np.float32)
    _, Y, _ = check(sdnn, oracle_mod, p, X=X)
    np.testing.assert_array_equal(Y, np.repeat(np.maximum(p.bias, 0)[:, None], N, 1))


def test_n_zero_is_noop(sdnn):
    p = synth.config_problem("c1")
    h = sdnn.Handle.from_problem(p)
    out = torch.full((p.M, 0), 1.0, device="cuda")
    h.spmm(torch.empty((p.K, 0), device="cuda"), None, out=out)


# ------------------------------------------------------------------ invariants (bitwise)
def test_permute_on_off_and_tilings_bitwise(sdnn):
    """Every kernel and tiling accumulates each row in ascending column order → identical Y (rows
    are not split here: split rows sum fixed pieces, see test_split_rows)."""
    p = synth.config_problem("c2_768x3072")
    X = p.x()
    ref, _ = run_gpu(sdnn, p, X, p.bias, 1, split_rows=False, split_k=False)
    for opts in [dict(permute=False), dict(panel_rows=8), dict(cta_panels=1), dict(k_chunk=8),
                 dict(k_chunk=96, panel_rows=4, cta_panels=2), dict(kernel="group"), dict(kernel="row"),
                 dict(kernel="group", permute=False), dict(kernel="group", cta_panels=3, k_chunk=16),
                 dict(kernel="group", group_sb=1), dict(kernel="group", group_sb=2), dict(kernel="group", group_sb=4),
                 dict(kernel="codegen"), dict(kernel="codegen", permute=False), dict(kernel="codegen", panel_rows=7),
                 dict(kernel="tmem"), dict(kernel="tmem", permute=False), dict(kernel="tmem8"),
                 dict(kernel="tmem8", permute=False)]:
        Y, _ = run_gpu(sdnn, p, X, p.bias, 1, split_rows=False, split_k=False, **opts)
        np.testing.assert_array_equal(Y, ref, err_msg=str(opts))


@pytest.mark.parametrize("key", ["c2_768x768", "c2_768x3072", "c2_3072x768"])
def test_split_rows(sdnn, oracle_mod, key):
    """Heavy log-normal rows split into pieces (row plan): parity with the oracle, deterministic,
    invariant to column shards and to the permutation (the pieces depend on the row only), close to
    the unsplit result, and capturable in a CUDA graph (stream-ordered workspace)."""
    p = synth.config_problem(key)
    X = p.x()
    worst, Y, h = check(sdnn, oracle_mod, p, kernel="row")
    assert h.info()["num_pieces"] > 0
    Y2, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    np.testing.assert_array_equal(Y, Y2)
    Ys, _ = run_gpu(sdnn, p, np.ascontiguousarray(X[:, 100:612]), p.bias, 1, handle=h)
    np.testing.assert_array_equal(Ys, Y[:, 100:612])
    Yp, _ = run_gpu(sdnn, p, X, p.bias, 1, kernel="row", permute=False)
    np.testing.assert_array_equal(Yp, Y)
    Yu, _ = run_gpu(sdnn, p, X, p.bias, 1, kernel="row", split_rows=False)
    Yo, S = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1, want_scale=True)[:2]
    assert_parity(Yu, Yo, S, "unsplit")
    Xd = torch.from_numpy(X).cuda()
    b = torch.from_numpy(p.bias).cuda()
    Yg = torch.empty((p.M, p.N), device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        h.spmm(Xd, b, act=1, out=Yg)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Yg.cpu().numpy(), Y)


def test_column_shards_bitwise(sdnn):
    p = synth.config_problem("c3_512x512")
    X = p.x()
    h = sdnn.Handle.from_problem(p, split_k=False)  # split-K slices depend on the grid, hence on N
    ref, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    for a, b in [(0, 4), (4, 1000), (1000, 1001), (1001, p.N)]:
        Y, _ = run_gpu(sdnn, p, np.ascontiguousarray(X[:, a:b]), p.bias, 1, handle=h)
        np.testing.assert_array_equal(Y, ref[:, a:b])


def test_repeat_bitwise_and_linearity(sdnn):
    p = synth.config_problem("c3_1024x512", act=0)
    X = p.x()
    h = sdnn.Handle.from_problem(p)
    Y1, _ = run_gpu(sdnn, p, X, None, 0, handle=h)
    Y2, _ = run_gpu(sdnn, p, X, None, 0, handle=h)
    np.testing.assert_array_equal(Y1, Y2)
    Y3, _ = run_gpu(sdnn, p, 2 * X, None, 0, handle=h)
    np.testing.assert_array_equal(Y3, 2 * Y1)


@pytest.mark.parametrize("kernel", ["row", "codegen", "tmem", "auto"])
def test_host_entry_point_matches_device(sdnn, kernel):
    p = synth.config_problem("c3_256x128")
    X = p.x()
    h = sdnn.Handle.from_problem(p, kernel=kernel, **({} if kernel == "codegen" else dict(split_k=False)))
    ref, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    for bc in (0, 512, 1000, 4, 2048):
        Y = h.spmm_host(X, p.bias, act=1, block_cols=bc)
        np.testing.assert_array_equal(Y, ref)


@pytest.mark.parametrize("kernel", ["row", "codegen", "tmem", "tmem8", "auto"])
def test_cuda_graph_capture(sdnn, kernel):
    p = synth.config_problem("c3_512x512")
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    X = torch.from_numpy(p.x()).cuda()
    b = torch.from_numpy(p.bias).cuda()
    Y = torch.empty((p.M, p.N), device="cuda")
    ref = h.spmm(X, b, act=1).clone()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        h.spmm(X, b, act=1, out=Y)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Y, ref)


def test_auto_takes_tmem_plan_when_it_fills_a_wave(sdnn):
    """kernel=auto keeps a TMEM plan beside the row plan (info alt_kernel = 4) and uses it when the
    call is on its fast path and fills one wave; either way the result equals the row kernel's."""
    p = synth.config_problem("c4_2048x512_s80")  # 35 row blocks × 25 N tiles ≥ 148 SMs / 2
    X = p.x()
    h = sdnn.Handle.from_problem(p)
    assert h.info()["alt_kernel"] == 4 and h.info()["kernel"] == 1
    Ya, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    Yr, _ = run_gpu(sdnn, p, X, p.bias, 1, kernel="row")
    np.testing.assert_array_equal(Ya, Yr)
    Xs = np.ascontiguousarray(X[:, :100])  # ragged: the row plan (split-K off: the bitwise order)
    Ya, _ = run_gpu(sdnn, p, Xs, p.bias, 1, handle=sdnn.Handle.from_problem(p, split_k=False))
    np.testing.assert_array_equal(Ya, Yr[:, :100])
    assert h.kernel_for(p.N) == 4 and h.kernel_for(102) == -1 and h.kernel_for(128) == 1  # 35·1·2 < 148


@pytest.mark.parametrize("M,K,sp", [(2048, 2048, 0.9), (4096, 1024, 0.7), (3072, 3072, 0.9)])
def test_auto_narrow_row_plan_for_small_grids(sdnn, oracle_mod, M, K, sp):
    """An auto handle whose row plan has few row blocks also keeps a narrow row plan (4-row panels,
    ≥ 64 row blocks, same permutation) for row-plan calls under one wave of CTAs (small N).  Same
    per-row accumulation order → bitwise equal to the row plan; oracle parity."""
    p = synth.make_problem(f"narrow{M}", M, K, 256, sp)
    h = sdnn.Handle.from_problem(p, split_k=False)
    info = h.info()
    assert info["narrow_row_blocks"] >= 64 and info["narrow_row_blocks"] > info["num_row_blocks"]
    # and the 16-row-block plan (narrow4) for N-tile-128 grids of one to three waves
    assert info["narrow4_row_blocks"] == (M + 15) // 16
    hr = sdnn.Handle.from_problem(p, kernel="row", split_k=False)
    assert hr.info()["narrow_row_blocks"] == 0 and hr.info()["narrow4_row_blocks"] == 0
    for N in (128, 256, 100):
        X = np.ascontiguousarray(p.x()[:, :N])
        Ya, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
        Yr, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=hr)
        np.testing.assert_array_equal(Ya, Yr)
        Yo, S = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1, want_scale=True)[:2]
        assert_parity(Ya, Yo, S, f"narrow N={N}")


@pytest.mark.parametrize("M,K,N,sp", [(3072, 3072, 128, 0.9), (4096, 4096, 128, 0.7), (2048, 2048, 256, 0.95),
                                      (3072, 3072, 200, 0.9)])
def test_auto_narrow4_with_split_k(sdnn, oracle_mod, M, K, N, sp):
    """Auto handles at N where the 16-row-block plan (narrow4) takes the call — with split-K where its
    grid leaves SMs under-filled (3072², N = 128: 192 CTAs of 5 warps → 2 slices), and N = 200
    (ragged tail tile): oracle parity and bitwise repeatability."""
    p = synth.make_problem(f"n4_{M}_{sp}", M, K, N, sp)
    h = sdnn.Handle.from_problem(p)
    assert h.info()["narrow4_row_blocks"] == (M + 15) // 16
    X = p.x()
    Y, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    Y2, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    np.testing.assert_array_equal(Y, Y2)
    Yo, S = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1, want_scale=True)[:2]
    assert_parity(Y, Yo, S, f"narrow4 {M}x{K} N={N}")


@pytest.mark.parametrize("M,K,N,sp,mask", [(512, 4096, 128, 0.9, "uniform"), (768, 3072, 128, 0.9, "uniform"),
                                            (768, 3072, 64, 0.9, "lognormal"), (256, 2048, 96, 0.8, "uniform")])
def test_split_k(sdnn, oracle_mod, M, K, N, sp, mask):
    """Row-kernel calls that leave the GPU under-filled split the K range over CTAs (partial sums reduced in slice
    order): oracle parity, deterministic (bitwise on repeat and in a CUDA graph), within rounding of
    the unsplit result, and SDNN_FLAG_NO_SPLIT_K turns it off."""
    p = synth.make_problem(f"sk{M}_{K}", M, K, N, sp, mask=mask)
    X = p.x()
    h = sdnn.Handle.from_problem(p, split_rows=False)
    Y, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    Y2, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    np.testing.assert_array_equal(Y, Y2)
    Yo, S = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1, want_scale=True)[:2]
    assert_parity(Y, Yo, S, "split-K")
    Yn, _ = run_gpu(sdnn, p, X, p.bias, 1, split_rows=False, split_k=False)
    assert_parity(Yn, Yo, S, "unsplit")
    assert not np.array_equal(Y, Yn)  # a different (slice-order) summation actually ran
    Xd, b = torch.from_numpy(X).cuda(), torch.from_numpy(p.bias).cuda()
    Yg = torch.empty((p.M, p.N), device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        h.spmm(Xd, b, act=1, out=Yg)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Yg.cpu().numpy(), Y)


@pytest.mark.parametrize("M,K,N,mask", [(768, 3072, 1024, "uniform"), (768, 3072, 512, "lognormal"), (512, 4096, 2048, "uniform")])
def test_tmem_split_k(sdnn, oracle_mod, M, K, N, mask):
    """Auto calls on the TMEM fast path with too few CTAs but a long K run the TMEM kernel over
    K-chunk slices (cut at even chunks) + the slice-ordered reduction: oracle parity, deterministic,
    CUDA-graph capturable; SDNN_FLAG_NO_SPLIT_K falls back to the row plan."""
    p = synth.make_problem(f"tsk{M}_{K}", M, K, N, 0.9, mask=mask)
    X = p.x()
    h = sdnn.Handle.from_problem(p)
    assert h.kernel_for(N, 256, 256) == 4  # the TMEM plan takes the call
    Y, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    Y2, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    np.testing.assert_array_equal(Y, Y2)
    Yo, S = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1, want_scale=True)[:2]
    assert_parity(Y, Yo, S, "TMEM split-K")
    hn = sdnn.Handle.from_problem(p, split_k=False)
    assert hn.kernel_for(N, 256, 256) != 4
    Xd, b = torch.from_numpy(X).cuda(), torch.from_numpy(p.bias).cuda()
    Yg = torch.empty((p.M, p.N), device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        h.spmm(Xd, b, act=1, out=Yg)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Yg.cpu().numpy(), Y)


@pytest.mark.parametrize("key,N", [("c2_768x3072", 1024), ("c3_512x512", 6272), ("c1", 128), ("narrow", 256)])
def test_tune(sdnn, oracle_mod, key, N):
    """sdnn_tune (per-matrix autotuning): the chosen path is kept for this N, its results match
    the oracle and repeat bitwise, and other N keep the automatic choice."""
    p = synth.make_problem("tn_nw", 2048, 1024, 256, 0.9) if key == "narrow" else synth.config_problem(key)
    X = np.ascontiguousarray(p.x_cols(0, N))
    h = sdnn.Handle.from_problem(p)
    auto_kernel = h.kernel_for(N // 2 * 2 - 4 if N > 8 else N, 256, 256)
    r = h.tune(torch.from_numpy(X).cuda())
    assert r["path"] in ("auto", "tmem", "row", "narrow", "narrow4") and r["us"] > 0
    if r["path"] != "auto":
        assert r["split_k"] in (1, 2, 4, 8) and h.kernel_for(N, 256, 256) == (4 if r["path"] == "tmem" else 1)
    Y, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    Y2, _ = run_gpu(sdnn, p, X, p.bias, 1, handle=h)
    np.testing.assert_array_equal(Y, Y2)
    Yo, S = oracle_mod.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1, want_scale=True)[:2]
    assert_parity(Y, Yo, S, f"tuned {r}")
    assert h.kernel_for(N // 2 * 2 - 4 if N > 8 else N, 256, 256) == auto_kernel  # other N: untouched


def test_get_permutation_and_info(sdnn, oracle_mod):
    p = synth.config_problem("c2_768x768")
    h = sdnn.Handle.from_problem(p)
    np.testing.assert_array_equal(h.permutation(), oracle_mod.alg1(p.row_ptr, p.col_idx, p.M, p.K))
    info = h.info()
    assert info["device"] == torch.cuda.current_device() and info["nnz"] == p.nnz and info["meta_bytes"] > 0


def test_errors(sdnn):
    p = synth.config_problem("c1")
    h = sdnn.Handle.from_problem(p)
    X = torch.zeros((p.K, 8), device="cuda")
    with pytest.raises(sdnn.SdnnError):
        h.spmm(X, None, act=5)
    st = sdnn._lib.sdnn_spmm(h._h, X.data_ptr(), -1, None, 1, X.data_ptr(), None)
    assert st == 1
    st = sdnn._lib.sdnn_spmm(h._h, X.data_ptr(), 8, None, 1, X.data_ptr(), None)  # Y aliases X
    assert st == 1


# ------------------------------------------------------------------ property-based shapes (hypothesis)
try:
    from hypothesis import given, settings, HealthCheck
    from hypothesis import strategies as st
except ImportError:  # pragma: no cover
    given = None

if given is not None:
    @pytest.mark.parametrize("kernel", ["auto", "row", "tmem", "tmem8", "tmemp"])
    @settings(max_examples=12, deadline=None, suppress_health_check=list(HealthCheck))
    @given(M=st.integers(1, 300), K=st.integers(1, 300), nq=st.integers(1, 6), ragged=st.booleans(),
           dens=st.sampled_from([0.0, 0.02, 0.1, 0.3, 1.0]), seed=st.integers(0, 2**31 - 1),
           mask=st.sampled_from(["uniform", "blocks4"]))
    def test_random_shapes(sdnn, oracle_mod, kernel, M, K, nq, ragged, dens, seed, mask):
        """Random M, K, density, N (multiples of 128 — the TMEM fast path — or ragged), uniform or
        aligned-1×4-run masks, every kernel: |Y − oracle| ≤ 1e-4·S."""
        rng = np.random.default_rng(seed)
        N = 128 * nq + (int(rng.integers(1, 128)) if ragged else 0)
        if mask == "blocks4":
            blk = rng.random((M, (K + 3) // 4)) < dens
            m = np.repeat(blk, 4, axis=1)[:, :K]
        else:
            m = rng.random((M, K)) < dens
        rp = np.zeros(M + 1, np.int32); rp[1:] = np.cumsum(m.sum(1))
        ci = np.nonzero(m)[1].astype(np.int32)
        v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
        v[v == 0] = 0.01
        b = (0.1 * rng.standard_normal(M)).astype(np.float32)
        p = synth.Problem("rand", M, K, N, 0, "x", rp, ci, v, b, 1, seed)
        X = rng.standard_normal((K, N)).astype(np.float32)
        check(sdnn, oracle_mod, p, X=X, act=int(seed % 2), kernel=kernel)


@pytest.mark.parametrize("K", [2, 64, 65, 128, 192, 256, 300, 448, 512])
@pytest.mark.parametrize("kernel,mask", [("auto", "uniform"), ("tmem", "blocks4")])
def test_short_k_many_items(sdnn, oracle_mod, K, kernel, mask):
    """Short K ranges (1-8 chunks of 64, odd and even counts) over >= 4 (row block, N tile) items per SM:
    the calls the launch rules may run on persistent TMEM-R CTAs.  Regression: with an odd chunk count
    the persistent pipeline's alternating TMEM halves disagreed with the half packed into the metadata
    from a CTA's second item on (found by tests/stress/fuzz.py); odd counts now launch one CTA per item."""
    M, N = 2274, 7808  # 10 row blocks x 61 N tiles = 610 items > 4 x 148 SMs
    rng = np.random.default_rng(1000 + K)
    if mask == "blocks4":
        m = np.repeat(rng.random((M, (K + 3) // 4)) < 0.15, 4, axis=1)[:, :K]
    else:
        m = rng.random((M, K)) < 0.1
    rp = np.zeros(M + 1, np.int32); rp[1:] = np.cumsum(m.sum(1))
    ci = np.nonzero(m)[1].astype(np.int32)
    v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
    v[v == 0] = 0.01
    b = (0.1 * rng.standard_normal(M)).astype(np.float32)
    p = synth.Problem("shortk", M, K, N, 0, "x", rp, ci, v, b, 1, K)
    X = rng.standard_normal((K, N)).astype(np.float32)
    _, Y, h = check(sdnn, oracle_mod, p, X=X, kernel=kernel)
    assert h.kernel_for(N) == 4
    # permuted output (the chained-layer form) through the same launch
    hp = sdnn.Handle.from_problem(p, kernel=kernel, permuted_output=True)
    perm = hp.permutation()
    Yp = hp.spmm(torch.from_numpy(X).cuda(), torch.from_numpy(np.ascontiguousarray(b[perm])).cuda(), act=1).cpu().numpy()
    np.testing.assert_array_equal(Yp, Y[perm])


if given is not None:
    @settings(max_examples=10, deadline=None, suppress_health_check=list(HealthCheck))
    @given(M=st.integers(16, 1500), K=st.integers(1024, 4096), n4=st.integers(1, 50), dens=st.sampled_from([0.02, 0.1, 0.2]),
           bias=st.booleans(), act=st.integers(0, 1), seed=st.integers(0, 2**31 - 1))
    def test_random_small_n_long_k(sdnn, oracle_mod, M, K, n4, dens, bias, act, seed):
        """Small N, long K, auto kernel: the narrow plan, V = 2 tiles and split-K (slice-ordered
        reduction, with / without bias and ReLU) against the oracle."""
        rng = np.random.default_rng(seed)
        N = 4 * n4
        m = rng.random((M, K)) < dens
        rp = np.zeros(M + 1, np.int32); rp[1:] = np.cumsum(m.sum(1))
        ci = np.nonzero(m)[1].astype(np.int32)
        v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
        v[v == 0] = 0.01
        b = (0.1 * rng.standard_normal(M)).astype(np.float32)
        p = synth.Problem("randk", M, K, N, 0, "x", rp, ci, v, b, act, seed)
        X = rng.standard_normal((K, N)).astype(np.float32)
        check(sdnn, oracle_mod, p, X=X, act=act, bias=b if bias else None)


@pytest.mark.parametrize("kernel", ["auto", "row", "tmem", "tmemp"])
def test_large_k_and_large_m(sdnn, oracle_mod, kernel):
    """K = 40 000 (625 TMEM chunks) and M = 20 000 (334 TMEM row blocks) at small N."""
    for M, K, N, dens in [(96, 40000, 256, 0.01), (20000, 64, 128, 0.05)]:
        p = synth.make_problem(f"big_{M}x{K}", M, K, N, 1 - dens, seed=M + K)
        check(sdnn, oracle_mod, p, kernel=kernel)


# ------------------------------------------------------------------ fused all-gather form (sdnn_spmm_multi)
@pytest.mark.parametrize("kernel", ["auto", "row", "tmem", "tmem8", "tmemp"])
@pytest.mark.parametrize("key,N", [("c3_512x512", 1024), ("c3_512x512", 1000), ("c2_768x768", 512), ("c1", 128)])
def test_spmm_multi_destinations(sdnn, key, N, kernel):
    """Y written to 3 buffers of leading dimension ldy at column offset col0 (the all-gather layout a
    rank writes into every peer's symmetric buffer): each equals the plain result, untouched elsewhere."""
    p = synth.config_problem(key, N=N)
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    X = torch.from_numpy(p.x()).cuda()
    b = torch.from_numpy(p.bias).cuda()
    ref = h.spmm(X, b, act=1).clone()
    col0, ldy = 256, N + 512
    bufs = [torch.full((p.M, ldy), -7.0, device="cuda") for _ in range(3)]
    h.spmm_multi(X, [t.data_ptr() for t in bufs], ldy, col0, bias=b, act=1)
    torch.cuda.synchronize()
    for t in bufs:
        assert torch.equal(t[:, col0:col0 + N], ref)
        assert bool((t[:, :col0] == -7.0).all()) and bool((t[:, col0 + N:] == -7.0).all())


def test_spmm_multi_errors(sdnn):
    p = synth.config_problem("c1")
    h = sdnn.Handle.from_problem(p)
    X = torch.zeros((p.K, 8), device="cuda")
    Y = torch.zeros((p.M, 8), device="cuda")
    with pytest.raises(sdnn.SdnnError):
        h.spmm_multi(X, [], 8, 0)
    with pytest.raises(sdnn.SdnnError):
        h.spmm_multi(X, [Y.data_ptr()] * 9, 8, 0)
    with pytest.raises(sdnn.SdnnError):
        h.spmm_multi(X, [Y.data_ptr()], 7, 0)  # ldy < col0 + N
