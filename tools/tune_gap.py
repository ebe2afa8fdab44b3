"""Where do the per-call rules leave time on the table?  Random shapes (M, K in [64, 4096], N a multiple
of 128 up to 8192, 70-98 % sparsity, uniform / 1x4-run / log-normal masks): the call timed through the
rules (auto), then after sdnn_tune picked the fastest path for that N; prints the shapes where the tuned
path wins by more than 10 % (a rule gap) and the geometric mean of auto / tuned.

  python tools/tune_gap.py --n 120 --seed 1 > gpurun_out/tune_gap.log
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, torch, iters=30):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / iters)
    return best


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=120)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_2101_07948_b200 as sdnn

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(args.seed)
    ratios, gaps = [], []
    for case in range(args.n):
        M, K = (int(np.exp(rng.uniform(np.log(64), np.log(4096)))) for _ in range(2))
        N = 128 * int(np.exp(rng.uniform(0, np.log(64))))
        sp = float(rng.choice([0.7, 0.8, 0.9, 0.95, 0.98]))
        mk = str(rng.choice(["uniform", "uniform", "blocks4", "lognormal"]))
        if mk == "blocks4":
            m = np.repeat(rng.random((M, (K + 3) // 4)) < 1 - sp, 4, axis=1)[:, :K]
        elif mk == "lognormal":
            m = rng.random((M, K)) < np.clip((1 - sp) * rng.lognormal(0.0, 1.0, size=(M, 1)), 0, 1)
        else:
            m = rng.random((M, K)) < 1 - sp
        rp = np.zeros(M + 1, np.int32)
        rp[1:] = np.cumsum(m.sum(1))
        ci = np.nonzero(m)[1].astype(np.int32)
        if ci.size == 0:
            continue
        v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
        h = sdnn.Handle(rp, ci, v, M, K)
        X = torch.randn((K, N), dtype=torch.float32, device=dev)
        b = torch.randn(M, dtype=torch.float32, device=dev)
        Y = torch.empty((M, N), dtype=torch.float32, device=dev)
        kid = h.kernel_for(N, X.data_ptr(), Y.data_ptr())
        t_auto = timed(lambda: h.spmm(X, b, act=1, out=Y), torch)
        t = h.tune(X, out=Y)
        t_tuned = timed(lambda: h.spmm(X, b, act=1, out=Y), torch)
        r = t_auto / t_tuned
        ratios.append(r)
        line = (f"M={M} K={K} N={N} sp={sp} {mk} nnz={ci.size} auto kernel {kid}: {t_auto:.1f} us -> tuned {t} {t_tuned:.1f} us "
                f"(x{r:.2f})")
        if r > 1.10:
            gaps.append(line)
        print(line, flush=True)
        h.close()
    g = float(np.exp(np.mean(np.log(ratios))))
    print(f"# {len(ratios)} shapes: geometric mean auto / tuned = {g:.3f}; {len(gaps)} shapes where the tuned path wins by > 10 %:")
    for ln in sorted(gaps, key=lambda s: -float(s.rsplit('(x', 1)[1][:-1])):
        print("#   " + ln)
    return 0


if __name__ == "__main__":
    sys.exit(main())
