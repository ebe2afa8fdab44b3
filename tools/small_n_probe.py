"""Probe the sweep's weakest points (low sparsity, small N: tools/sweep.py) — auto choice, the tuner's
choice, and row-plan geometries — to see where the time goes.
usage: python tools/small_n_probe.py [--points 4096x4096:0.7:128,2048x2048:0.7:512]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tools"))
from sweep import graph_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", default="4096x4096:0.7:128,4096x4096:0.8:128,2048x2048:0.7:512,2048x2048:0.7:128")
    ap.add_argument("--geoms", default="0x0,4x4,4x8,8x4,8x8,16x4,2x8")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    for pt in a.points.split(","):
        mk, sp, n = pt.split(":")
        M, K = (int(v) for v in mk.split("x"))
        N = int(n)
        p = synth.make_problem(pt, M, K, N, float(sp))
        X = torch.randn((K, N), device="cuda")
        b = torch.from_numpy(p.bias).cuda()
        Y = torch.empty((M, N), device="cuda")
        h = sdnn.Handle.from_problem(p)
        t = graph_time(lambda: h.spmm(X, b, act=1, out=Y), a.reps)
        flop = 2 * p.nnz * N
        print(f"{pt:22s} auto      kernel={h.kernel_for(N, X.data_ptr(), Y.data_ptr())} {t:8.2f} us {flop / t / 1e6:6.2f} TF", flush=True)
        r = h.tune(X, out=Y)
        t = graph_time(lambda: h.spmm(X, b, act=1, out=Y), a.reps)
        print(f"{pt:22s} tuned     {r} {t:8.2f} us {flop / t / 1e6:6.2f} TF", flush=True)
        h.close()
        for g in a.geoms.split(","):
            pr, cp = (int(v) for v in g.split("x"))
            for ks in (True, False):
                opts = {"kernel": "row", "split_k": ks}
                if pr:
                    opts.update(panel_rows=pr, cta_panels=cp)
                try:
                    h = sdnn.Handle.from_problem(p, **opts)
                except Exception as e:  # noqa: BLE001
                    print(f"{pt:22s} row {g} ks={ks}: {e}")
                    continue
                t = graph_time(lambda: h.spmm(X, b, act=1, out=Y), a.reps)
                inf = h.info()
                print(f"{pt:22s} row {g:5s} ks={int(ks)} blocks={inf.get('num_row_blocks')} chunks={inf.get('num_chunks')} "
                      f"{t:8.2f} us {flop / t / 1e6:6.2f} TF", flush=True)
                h.close()


if __name__ == "__main__":
    main()
