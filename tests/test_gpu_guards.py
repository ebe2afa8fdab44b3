"""Out-of-bounds write guards on every kernel path (compute-sanitizer is not available on the GPU
pool, so — SURVEY §4 test layer 4 by other means): each output lives inside a larger buffer whose
guard zones before and after hold a sentinel; after the call the guards must be untouched and the
output must match the oracle.  Covers the row kernel (V = 2/4/8, generic ragged tail), split rows,
split-K, the narrow plan, TMEM V = 4/8 (incl. 1×4 runs and the ragged fallback), the group kernel,
multi-destination stores, the host-buffer pipeline and both sparse-convolution forms."""
import numpy as np
import pytest

import sdnn_synth as synth
from oracle import conv as oconv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
G = 4096  # guard floats on each side (16-byte multiple keeps the output aligned)
SENT = 12345.0


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


def guarded(shape, extra=0):
    n = int(np.prod(shape))
    buf = torch.full((G + n + G + extra,), SENT, device="cuda")
    return buf, buf[G + extra:G + extra + n].view(*shape)


def assert_guards(buf, n, extra=0):
    b = buf.cpu().numpy()
    assert np.all(b[:G + extra] == SENT) and np.all(b[G + extra + n:] == SENT), "write outside the output"


def parity(Y, Yo, S):
    zero = S == 0
    assert np.all(Y[zero] == Yo[zero])
    err = np.abs(Y.astype(np.float64) - Yo) / np.where(zero, 1.0, S)
    assert float(err.max()) <= 1e-4, float(err.max())


CASES = [  # (problem, N, handle options)
    ("c1", 128, {}), ("c1", 100, {}), ("c1", 512, dict(kernel="tmem")), ("c1", 1024, dict(kernel="tmem8")),
    ("c1", 96, dict(kernel="tmem")), ("c1", 256, dict(kernel="group")), ("c1", 1000, dict(kernel="row", cta_panels=1)),
    ("lognormal", 64, dict(kernel="row")), ("splitk", 96, {}), ("block4", 512, dict(kernel="tmem")),
    ("c1", 512, dict(kernel="tmemp")), ("c1", 96, dict(kernel="tmemp")),
    ("narrow", 128, {}), ("narrow", 68, {}),
]


def problem(key):
    if key == "c1":
        return synth.config_problem("c1", N=1024)
    if key == "lognormal":
        return synth.make_problem("g_lg", 384, 512, 64, 0.9, mask="lognormal")
    if key == "splitk":
        return synth.make_problem("g_sk", 256, 2048, 96, 0.8)
    if key == "block4":
        return synth.make_problem("g_b4", 240, 256, 512, 0.8, mask="block4")
    return synth.make_problem("g_nw", 2048, 512, 128, 0.9)


@pytest.mark.parametrize("key,N,opts", CASES)
def test_spmm_guarded(sdnn, oracle_mod, key, N, opts):
    p = problem(key)
    X = np.ascontiguousarray(p.x_cols(0, N))
    h = sdnn.Handle.from_problem(p, **opts)
    for extra in (0, 1):  # extra = 1 float: a 4-byte-aligned (not 16) output takes the generic path
        buf, Y = guarded((p.M, N), extra)
        h.spmm(torch.from_numpy(X).cuda(), torch.from_numpy(p.bias).cuda(), act=1, out=Y)
        torch.cuda.synchronize()
        assert_guards(buf, p.M * N, extra)
        Yo, S = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
        parity(Y.cpu().numpy(), Yo, S)


@pytest.mark.parametrize("kernel,N", [("tmem", 512), ("row", 96), ("auto", 1024)])
def test_spmm_multi_guarded(sdnn, oracle_mod, kernel, N):
    p = synth.config_problem("c1", N=1024)
    X = np.ascontiguousarray(p.x_cols(0, N))
    h = sdnn.Handle.from_problem(p, kernel=kernel)
    ld, col0 = N + 8, 4
    bufs = [guarded((p.M, ld)) for _ in range(2)]
    h.spmm_multi(torch.from_numpy(X).cuda(), [Y.data_ptr() for _, Y in bufs], ldy=ld, col0=col0,
                 bias=torch.from_numpy(p.bias).cuda(), act=1)
    torch.cuda.synchronize()
    Yo, S = oracle_mod.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    for buf, Y in bufs:
        assert_guards(buf, p.M * ld)
        Yc = Y.cpu().numpy()
        assert np.all(Yc[:, :col0] == SENT) and np.all(Yc[:, col0 + N:] == SENT)  # untouched columns
        parity(Yc[:, col0:col0 + N], Yo, S)


def test_conv_guarded(sdnn):
    for cp in (synth.make_conv_problem("g_c1", 48, 40, 7, 7, 2, 0.9),
               synth.make_conv_problem("g_c2", 16, 8, 9, 11, 1, 0.8, stride=2)):
        h = sdnn.Handle(cp.row_ptr, cp.col_idx, cp.vals, cp.OC, cp.K, split_rows=False)
        Xc = cp.x()
        buf, Y = guarded((cp.OC, cp.B, cp.Ho, cp.Wo))
        h.conv2d(torch.from_numpy(Xc).cuda(), cp.FY, cp.FX, cp.pad, cp.stride, torch.from_numpy(cp.bias).cuda(),
                 act=1, out=Y)
        torch.cuda.synchronize()
        assert_guards(buf, Y.numel())
        Yo, S = oconv.conv2d(cp.row_ptr, cp.col_idx, cp.vals, cp.OC, cp.IC, cp.FY, cp.FX, Xc, cp.pad, cp.stride,
                             cp.bias, 1)
        parity(Y.cpu().numpy(), Yo, S)
