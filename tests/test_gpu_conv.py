"""Sparse k×k convolution through the C ABI (sdnn_conv2d)
against the convolution oracle (oracle/conv.py, the definition in fp64) element by element with the
north_star tolerance |Y − Y_oracle| ≤ 1e-4·S, S = Σ|w||x| + |b| (exact where S = 0)."""
import numpy as np
import pytest

import sdnn_synth as synth
from oracle import conv as oconv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def sdnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_07948_b200 as m
    return m


def run(sdnn, p, **hopts):
    h = sdnn.Handle.for_conv(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, p.FY, p.FX, **hopts)
    X = p.x()
    b = None if p.bias is None else torch.from_numpy(p.bias).cuda()
    Y = h.conv2d(torch.from_numpy(X).cuda(), p.FY, p.FX, p.pad, p.stride, b, act=p.act).cpu().numpy()
    Yo, S = oconv.conv2d(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, p.FY, p.FX, X, p.pad, p.stride, p.bias, p.act)
    zero = S == 0
    assert np.all(Y[zero] == Yo[zero])
    err = np.abs(Y.astype(np.float64) - Yo) / np.where(zero, 1.0, S)
    assert float(err.max()) <= TOL, float(err.max())
    return Y, h


# the paper's suite: IC/OC 32..256, images 7/14/28/56, 3×3 pad 1, 90 / 95 %; batch 1-4
@pytest.mark.parametrize("OC,IC,HW,B,sp", [(32, 32, 7, 4, 0.9), (64, 128, 14, 2, 0.95), (128, 64, 28, 1, 0.9),
                                            (256, 256, 14, 1, 0.95), (64, 32, 56, 1, 0.9), (256, 128, 7, 3, 0.9)])
def test_conv_suite_parity(sdnn, OC, IC, HW, B, sp):
    run(sdnn, synth.make_conv_problem(f"cs{OC}_{IC}_{HW}", OC, IC, HW, HW, B, sp))


@pytest.mark.parametrize("FY,FX,pad,stride", [(3, 3, 0, 1), (3, 3, 1, 2), (5, 5, 2, 1), (1, 1, 0, 1), (1, 3, 0, 1),
                                                 (3, 5, 2, 2)])  # 3×5: a whole-channel chunk (120) does not fit → the library's own chunks
def test_conv_shapes(sdnn, FY, FX, pad, stride):
    run(sdnn, synth.make_conv_problem(f"sh{FY}{FX}{pad}{stride}", 48, 24, 13, 11, 2, 0.85, FY=FY, FX=FX, pad=pad,
                                      stride=stride))


def test_conv_no_bias_no_act_and_row_plans(sdnn):
    p = synth.make_conv_problem("nb", 40, 16, 9, 9, 2, 0.8, bias=False, act=0)
    Y1, _ = run(sdnn, p)
    Y2, _ = run(sdnn, p, kernel="row", panel_rows=8, cta_panels=4)
    np.testing.assert_array_equal(Y1, Y2)  # same per-row accumulation order


def test_one_by_one_conv_equals_spmm(sdnn):
    p = synth.make_conv_problem("c11", 64, 48, 10, 12, 2, 0.9, FY=1, FX=1, pad=0)
    Yc, h = run(sdnn, p, split_k=False)  # bitwise: the same (unsplit) summation order on both sides
    X = torch.from_numpy(p.x().reshape(p.IC, -1).copy()).cuda()
    Ys = h.spmm(X, torch.from_numpy(p.bias).cuda(), act=1).cpu().numpy()
    np.testing.assert_array_equal(Yc.reshape(p.OC, -1), Ys)


def test_conv_errors(sdnn):
    p = synth.make_conv_problem("err", 16, 8, 6, 6, 1, 0.8)
    h = sdnn.Handle(p.row_ptr, p.col_idx, p.vals, p.OC, p.K, split_rows=False)
    X = torch.from_numpy(p.x()).cuda()
    with pytest.raises(sdnn.SdnnError):
        h.conv2d(X[:4].contiguous(), 3, 3, 1, 1)  # IC·9 != K
    ht = sdnn.Handle(p.row_ptr, p.col_idx, p.vals, p.OC, p.K, kernel="tmem")
    with pytest.raises(sdnn.SdnnError):
        ht.conv2d(X, 3, 3, 1, 1)


def test_conv_split_k(sdnn):
    """Small images with many input channels split the K range over CTAs (partial sums reduced in
    slice order): oracle parity, deterministic, and SDNN_FLAG_NO_SPLIT_K gives the sequential order."""
    p = synth.make_conv_problem("csk", 256, 256, 7, 7, 1, 0.9)
    Y1, h = run(sdnn, p)
    Y2, _ = run(sdnn, p)
    np.testing.assert_array_equal(Y1, Y2)
    Yn, _ = run(sdnn, p, split_k=False)
    assert not np.array_equal(Y1, Yn)  # the split path actually ran


@pytest.mark.parametrize("C,HW", [(128, 14), (64, 7)])
def test_conv_tune(sdnn, C, HW):
    """sdnn_conv2d_tune keeps a choice per geometry (pixels per lane of the patch form, or −2: the
    explicit form, im2col + TMEM-R SpMM); tuned results match the oracle."""
    p = synth.make_conv_problem(f"ctn{C}_{HW}", C, C, HW, HW, 4, 0.9)
    h = sdnn.Handle.for_conv(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3)
    r = h.conv2d_tune(torch.from_numpy(p.x()).cuda())
    assert r["pixels"] in (-2, 0, 2, 4) and r["us"] > 0
    Xc = p.x()
    Y = h.conv2d(torch.from_numpy(Xc).cuda(), 3, 3, 1, 1, torch.from_numpy(p.bias).cuda(), act=1).cpu().numpy()
    Yo, S = oconv.conv2d(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3, Xc, 1, 1, p.bias, 1)
    err = np.abs(Y.astype(np.float64) - Yo) / np.where(S == 0, 1.0, S)
    assert float(err.max()) <= TOL



@pytest.mark.parametrize("OC,IC,HW,B,sp", [(512, 128, 14, 8, 0.9), (480, 64, 28, 2, 0.8), (256, 256, 14, 8, 0.9)])
def test_conv_explicit_form(sdnn, OC, IC, HW, B, sp):
    """Layers with ≥ 480 filters take the explicit form (Xv = the virtual operand written out by
    im2col_kernel, then the TMEM-R SpMM of the handle's TMEM plan); smaller ones can get it from the
    tuner: oracle parity either way."""
    p = synth.make_conv_problem(f"ex{OC}_{IC}_{HW}", OC, IC, HW, HW, B, sp)
    Y, h = run(sdnn, p)
    X = torch.from_numpy(p.x()).cuda()
    r = h.conv2d_tune(X, p.FY, p.FX, p.pad, p.stride)
    assert r["pixels"] in (-2, 0, 2, 4)
    run_again = h.conv2d(X, p.FY, p.FX, p.pad, p.stride, torch.from_numpy(p.bias).cuda(), act=p.act).cpu().numpy()
    Yo, S = oconv.conv2d(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, p.FY, p.FX, p.x(), p.pad, p.stride, p.bias, p.act)
    err = np.abs(run_again.astype(np.float64) - Yo) / np.where(S == 0, 1.0, S)
    assert float(err.max()) <= TOL
