"""Extreme shapes against the oracle on a GPU (the ends of every index range the kernels and the planner
use): very tall / very wide W, one row / one column, K beyond 16-bit columns, M beyond the reduction
kernels' gridDim.y, N = 1, N beyond 2^20, a fully dense and an almost empty W, Y beyond 2^31 elements
(sampled columns).  One line per case; exit code 1 on any failure.

  python tests/stress/extreme.py > gpurun_out/extreme.log
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (the checker; this tool is test infrastructure)


def csr_random(rng, M, K, nnz_per_row):
    """About nnz_per_row nonzeros per row at distinct random columns (memory-light for huge M·K)."""
    counts = np.minimum(K, rng.poisson(nnz_per_row, size=M)).astype(np.int64)
    rp = np.zeros(M + 1, np.int32)
    rp[1:] = np.cumsum(counts)
    ci = np.empty(int(rp[-1]), np.int32)
    for r in range(M):
        n = int(counts[r])
        if n:
            ci[rp[r]:rp[r + 1]] = np.sort(rng.choice(K, size=n, replace=False))
    v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
    v[v == 0] = 0.01
    return rp, ci, v


def main() -> int:
    import torch
    import paper_2101_07948_b200 as sdnn

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    cases = [  # (name, M, K, N, nnz per row, options)
        ("tall M=300000 (beyond gridDim.y)", 300000, 64, 128, 4, {"permute": False}),
        ("tall, split-K tuned path", 70000, 2048, 64, 6, {"tune": True, "permute": False}),
        ("wide K=200000 (beyond 16-bit columns)", 64, 200000, 256, 300, {}),
        ("wide K, TMEM", 512, 70000, 1024, 50, {"kernel": "tmem"}),
        ("one row", 1, 5000, 4096, 700, {}),
        ("one column of W", 5000, 1, 4096, 1, {}),
        ("N = 1", 3000, 3000, 1, 30, {}),
        ("N = 3, tall", 100000, 100, 3, 5, {"permute": False}),
        ("N = 2^20 + 4, small W", 32, 32, (1 << 20) + 4, 4, {}),
        ("dense 600x600", 600, 600, 2048, 600, {}),
        ("dense 600x600 TMEM", 600, 600, 2048, 600, {"kernel": "tmem"}),
        ("almost empty", 4096, 4096, 4096, 0.01, {}),
        ("Y > 2^31 elements (sampled)", 40000, 64, 65536, 3, {"sample": 64, "permute": False}),
    ]
    fails = 0
    for name, M, K, N, npr, opt in cases:
        try:
            rp, ci, v = csr_random(rng, M, K, npr)
            b = (0.1 * rng.standard_normal(M)).astype(np.float32)
            hopts = {k: opt[k] for k in ("kernel", "permute") if k in opt}  # Algorithm 1 is O(M^2)-ish: off for the tall cases
            h = sdnn.Handle(rp, ci, v, M, K, **hopts)
            gen = torch.Generator(device=dev)
            gen.manual_seed(1)
            Xd = torch.randn((K, N), dtype=torch.float32, device=dev, generator=gen)
            bd = torch.from_numpy(b).to(dev)
            if opt.get("tune"):
                h.tune(Xd)
            Y = h.spmm(Xd, bd, act=1)
            torch.cuda.synchronize()
            if "sample" in opt:
                cols = np.unique(np.concatenate([[0, 1, N - 2, N - 1], rng.integers(0, N, opt["sample"])]))
                ct = torch.from_numpy(cols).to(dev)
                Xs, Ys = Xd[:, ct].cpu().numpy(), Y[:, ct].cpu().numpy()
            else:
                Xs, Ys = Xd.cpu().numpy(), Y.cpu().numpy()
            Yo, S, _ = oracle.spmm_omp(rp, ci, v, M, K, np.ascontiguousarray(Xs), b, act=1, want_scale=True)
            e = np.abs(Ys.astype(np.float64) - Yo) / np.where(S > 0, S, 1.0)
            ok = np.isfinite(Ys).all() and float(e.max(initial=0.0)) <= 1e-4 and np.all(Ys[S == 0] == Yo[S == 0])
            Y2 = h.spmm(Xd, bd, act=1)
            ok2 = bool(torch.equal(Y, Y2))
            print(f"{name}: M={M} K={K} N={N} nnz={ci.size} kernel_id={h.kernel_for(N, Xd.data_ptr())} "
                  f"max err/S {e.max(initial=0.0):.2e} -> {'ok' if ok and ok2 else 'FAIL'}{'' if ok2 else ' (repeat differs)'}", flush=True)
            fails += 0 if (ok and ok2) else 1
            h.close()
            del Xd, Y, Y2
            torch.cuda.empty_cache()
        except Exception as e:  # noqa: BLE001
            print(f"{name}: FAIL exception {type(e).__name__}: {e}", flush=True)
            fails += 1
    print(f"# {len(cases)} cases, {fails} failed")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
