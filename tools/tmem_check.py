"""Quick check of a kernel variant against the row kernel (bitwise) and the oracle (tolerance), plus
c5 timing.  usage: python tools/tmem_check.py [--kernel tmem] [--configs c1,c2_768x768,...] [--c5]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SDNN_PKG_DIR"):
    sys.path.insert(0, os.environ["SDNN_PKG_DIR"])

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="tmem")
    ap.add_argument("--configs", default=",".join(k for k in synth.CONFIGS if k != "c5"))
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    oracle.build()
    for key in a.configs.split(","):
        if not key:
            continue
        p = synth.config_problem(key)
        X = p.x()
        Xd = torch.from_numpy(X).cuda()
        b = torch.from_numpy(p.bias).cuda()
        hr = sdnn.Handle.from_problem(p, kernel="row")
        hk = sdnn.Handle.from_problem(p, kernel=a.kernel)
        Yr = hr.spmm(Xd, b, act=p.act).cpu().numpy()
        Yk = hk.spmm(Xd, b, act=p.act).cpu().numpy()
        Yo, S, _ = oracle.spmm_omp(p.row_ptr, p.col_idx, p.vals, p.M, p.K, X, p.bias, act=p.act, want_scale=True)
        err = np.abs(Yk.astype(np.float64) - Yo) / np.where(S > 0, S, 1.0)
        ts = {}
        for name, h in (("row", hr), (a.kernel, hk)):
            Y = torch.empty((p.M, p.N), device="cuda")
            for _ in range(3):
                h.spmm(Xd, b, act=p.act, out=Y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                h.spmm(Xd, b, act=p.act, out=Y)
            e1.record()
            torch.cuda.synchronize()
            ts[name] = e0.elapsed_time(e1) / a.iters * 1e3
        fl = 2 * p.nnz * p.N
        print(f"{key:18s} bitwise_vs_row={np.array_equal(Yr, Yk)} max_err/S={err.max():.2e} "
              f"row {ts['row']:8.1f} us ({fl / ts['row'] / 1e6:7.2f} TF)  {a.kernel} {ts[a.kernel]:8.1f} us "
              f"({fl / ts[a.kernel] / 1e6:7.2f} TF)", flush=True)
    if a.c5:
        p = synth.config_problem("c5")
        X = torch.empty((p.K, p.N), dtype=torch.float32, device="cuda")
        for bl in range((p.N + synth.X_BLOCK - 1) // synth.X_BLOCK):
            blk = torch.from_numpy(p.x_block(bl))
            X[:, bl * synth.X_BLOCK:bl * synth.X_BLOCK + blk.shape[1]].copy_(blk)
        b = torch.from_numpy(p.bias).cuda()
        res = {}
        for name in ("row", a.kernel):
            t0 = time.time()
            h = sdnn.Handle.from_problem(p, kernel=name)
            prep = time.time() - t0
            Y = torch.empty((p.M, p.N), device="cuda")
            h.spmm(X, b, act=1, out=Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                h.spmm(X, b, act=1, out=Y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            res[name] = Y[:, :8192].cpu().numpy()
            print(f"c5 {name:6s} prep {prep:.2f}s  {ms:8.2f} ms  {2 * p.nnz * p.N / ms / 1e9:7.2f} TF", flush=True)
            del Y
        print("c5 bitwise (first 8192 cols):", np.array_equal(res["row"], res[a.kernel]))


if __name__ == "__main__":
    main()
