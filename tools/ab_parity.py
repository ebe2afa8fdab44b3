"""Parity of one build (SDNN_PKG_DIR=ab/X) of the TMEM kernel against the oracle on the BASELINE
configs (c5 on 8192 columns): prints max |Y - Y_oracle| / S per config.  Experiments only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SDNN_PKG_DIR"):
    sys.path.insert(0, os.environ["SDNN_PKG_DIR"])
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402

worst = 0.0
for key in list(synth.CONFIGS):
    p = synth.config_problem(key, N=8192 if key == "c5" else None)
    N = p.N - p.N % 128 or 128
    X = p.x_cols(0, N) if key == "c5" else p.x()[:, :N]
    X = np.ascontiguousarray(X)
    h = sdnn.Handle.from_problem(p, kernel=os.environ.get("KERNEL", "tmem"))
    Y = h.spmm(torch.from_numpy(X).cuda(), torch.from_numpy(p.bias).cuda(), act=1).cpu().numpy()
    Yo, S = oracle.spmm(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=1)
    err = np.abs(Y.astype(np.float64) - Yo) / np.where(S > 0, S, 1.0)
    ok = err.max() <= 1e-4 and np.all(Y[S == 0] == Yo[S == 0])
    worst = max(worst, float(err.max()))
    print(f"{key:18s} N={N:6d} max err/S {err.max():.2e} {'ok' if ok else 'FAIL'}", flush=True)
print("worst", worst)
