"""Sparse convolution oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:148 (§3.2.3): "the sparse convolution is treated as an SpMM where the sparse matrix is
the filters treated as an OC by IC × Fx × Fy matrix ... The dense matrix is a virtual matrix that is
realized on the fly from the input dense activations with the proper offsets".  The oracle does not
follow that lowering: it is the plain definition of a 2-D cross-correlation with zero padding,

    Y[oc, b, oy, ox] = act( Σ_{ic, fy, fx} W[oc, ic, fy, fx] · Xpad[ic, b, oy·s + fy, ox·s + fx] + bias[oc] )

in fp64, rounded once to fp32 (as the SpMM oracle), with the error scale
S = Σ |W|·|Xpad| + |bias| (reading C9).  W is rebuilt densely from the CSR of the OC × (IC·FY·FX)
matrix (column (ic·FY + fy)·FX + fx).  One numpy contraction per filter tap.
Pinned by tests/test_conv_oracle.py (SPEC S:258 worked example, center-tap and 1×1 closed forms,
scipy correlate2d, pure-Python brute force).
"""
from __future__ import annotations

import numpy as np


def dense_filters(row_ptr, col_idx, vals, OC: int, IC: int, FY: int, FX: int) -> np.ndarray:
    Wd = np.zeros((OC, IC * FY * FX), np.float64)
    rows = np.repeat(np.arange(OC), np.diff(np.asarray(row_ptr, np.int64)))
    Wd[rows, np.asarray(col_idx, np.int64)] = np.asarray(vals, np.float64)
    return Wd.reshape(OC, IC, FY, FX)


def conv2d(row_ptr, col_idx, vals, OC: int, IC: int, FY: int, FX: int, X: np.ndarray, pad: int, stride: int,
           bias=None, act: int = 1):
    """X: [IC][B][H][W] float32.  Returns (Y float32 [OC][B][Ho][Wo], S float64 same shape)."""
    Wt = dense_filters(row_ptr, col_idx, vals, OC, IC, FY, FX)
    IC_, B, H, W = X.shape
    assert IC_ == IC
    Ho = (H + 2 * pad - FY) // stride + 1
    Wo = (W + 2 * pad - FX) // stride + 1
    Xp = np.zeros((IC, B, H + 2 * pad, W + 2 * pad), np.float64)
    Xp[:, :, pad:pad + H, pad:pad + W] = X
    acc = np.zeros((OC, B, Ho, Wo), np.float64)
    S = np.zeros((OC, B, Ho, Wo), np.float64)
    for fy in range(FY):
        for fx in range(FX):
            win = Xp[:, :, fy:fy + stride * (Ho - 1) + 1:stride, fx:fx + stride * (Wo - 1) + 1:stride]
            acc += np.einsum("oi,ibhw->obhw", Wt[:, :, fy, fx], win)
            S += np.einsum("oi,ibhw->obhw", np.abs(Wt[:, :, fy, fx]), np.abs(win))
    if bias is not None:
        b = np.asarray(bias, np.float64)[:, None, None, None]
        acc += b
        S += np.abs(b)
    if act == 1:
        acc = np.where(acc > 0.0, acc, 0.0)
    return acc.astype(np.float32), S
