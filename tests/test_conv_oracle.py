"""Pins for the sparse-convolution oracle (oracle/conv.py).  Each pin
is independent of the oracle's own formula: a printed worked example, closed forms, scipy's
correlate2d, the SpMM oracle (C) for 1×1 filters, and a pure-Python brute force on tiny inputs."""
import numpy as np
import pytest
from scipy.signal import correlate2d

import oracle
from oracle import conv as oconv
import sdnn_synth as synth


def csr_of(Wd):
    """CSR of the OC × (IC·FY·FX) matrix of a dense filter tensor (ic-major, then fy, then fx)."""
    OC = Wd.shape[0]
    M = Wd.reshape(OC, -1)
    rp = np.zeros(OC + 1, np.int32)
    cols, vals = [], []
    for r in range(OC):
        nz = np.nonzero(M[r])[0]
        cols.append(nz)
        vals.append(M[r, nz])
        rp[r + 1] = rp[r] + len(nz)
    return rp, np.concatenate(cols).astype(np.int32), np.concatenate(vals).astype(np.float32)


def test_spec_worked_example():
    # 3×3 all-ones single-channel filter, 3×3 all-ones image, pad 1
    rp, ci, v = csr_of(np.ones((1, 1, 3, 3), np.float32))
    Y, S = oconv.conv2d(rp, ci, v, 1, 1, 3, 3, np.ones((1, 1, 3, 3), np.float32), pad=1, stride=1, act=0)
    np.testing.assert_array_equal(Y[0, 0], [[4, 6, 4], [6, 9, 6], [4, 6, 4]])
    np.testing.assert_array_equal(S[0, 0], [[4, 6, 4], [6, 9, 6], [4, 6, 4]])


def test_center_tap_is_scaled_identity():
    c = np.float32(0.75)
    Wd = np.zeros((1, 1, 3, 3), np.float32)
    Wd[0, 0, 1, 1] = c
    X = np.random.default_rng(0).standard_normal((1, 2, 5, 7)).astype(np.float32)
    Y, _ = oconv.conv2d(*csr_of(Wd), 1, 1, 3, 3, X, pad=1, stride=1, act=0)
    np.testing.assert_array_equal(Y, (np.float64(c) * X).astype(np.float32))


def test_single_channel_matches_scipy_correlate2d():
    rng = np.random.default_rng(1)
    Wd = rng.standard_normal((1, 1, 3, 3)).astype(np.float32)
    X = rng.standard_normal((1, 1, 9, 11)).astype(np.float32)
    Y, _ = oconv.conv2d(*csr_of(Wd), 1, 1, 3, 3, X, pad=1, stride=1, act=0)
    ref = correlate2d(X[0, 0].astype(np.float64), Wd[0, 0].astype(np.float64), mode="same")
    np.testing.assert_allclose(Y[0, 0], ref.astype(np.float32), rtol=1e-6, atol=1e-6)


def test_one_by_one_is_the_spmm_oracle():
    p = synth.make_conv_problem("c1x1", 24, 16, 5, 6, 2, 0.8, FY=1, FX=1, pad=0)
    X = p.x()
    Y, S = oconv.conv2d(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 1, 1, X, 0, 1, p.bias, act=1)
    Ys, Ss = oracle.spmm(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, X.reshape(p.IC, -1), p.bias, act=1)
    np.testing.assert_array_equal(Y.reshape(p.OC, -1), Ys)
    np.testing.assert_allclose(S.reshape(p.OC, -1), Ss, rtol=1e-12)


@pytest.mark.parametrize("stride,pad,FY,FX", [(1, 1, 3, 3), (2, 1, 3, 3), (1, 0, 2, 3), (2, 2, 3, 3)])
def test_brute_force_tiny(stride, pad, FY, FX):
    p = synth.make_conv_problem(f"bf{stride}{pad}{FY}{FX}", 3, 2, 5, 6, 2, 0.5, FY=FY, FX=FX, pad=pad, stride=stride)
    X = p.x()
    Y, S = oconv.conv2d(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, FY, FX, X, pad, stride, p.bias, act=1)
    Wd = np.zeros((p.OC, p.IC * FY * FX))
    for r in range(p.OC):
        for q in range(p.row_ptr[r], p.row_ptr[r + 1]):
            Wd[r, p.col_idx[q]] = p.vals[q]
    Ho, Wo = p.Ho, p.Wo
    assert Y.shape == (p.OC, p.B, Ho, Wo)
    for oc in range(p.OC):
        for b in range(p.B):
            for oy in range(Ho):
                for ox in range(Wo):
                    s = 0.0
                    for ic in range(p.IC):
                        for fy in range(FY):
                            for fx in range(FX):
                                y, x = oy * stride + fy - pad, ox * stride + fx - pad
                                if 0 <= y < p.H and 0 <= x < p.W:
                                    s += Wd[oc, (ic * FY + fy) * FX + fx] * float(X[ic, b, y, x])
                    s += float(p.bias[oc])
                    assert Y[oc, b, oy, ox] == np.float32(max(s, 0.0)) or abs(Y[oc, b, oy, ox] - max(s, 0.0)) <= 1e-6 * S[oc, b, oy, ox]


def test_linearity():
    p = synth.make_conv_problem("lin", 8, 4, 6, 6, 1, 0.7, bias=False)
    X = p.x()
    Y1, S1 = oconv.conv2d(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3, X, 1, 1, None, act=0)
    Y2, _ = oconv.conv2d(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3, (2 * X).astype(np.float32), 1, 1, None, act=0)
    np.testing.assert_allclose(Y2, 2 * Y1, rtol=0, atol=1e-6 * S1.max())
