"""Randomised stress of the other entry points against the oracle on a GPU (companion of tests/stress/fuzz.py):
sdnn_conv2d (random geometry: 1x1..5x5, stride 1-2, pad 0-2, ragged images, with / without
sdnn_conv2d_tune), sdnn_spmm_host (random block sizes), Chain (2-3 layers with the permutation carried
across layers) and sdnn_spmm_multi (several destinations, leading dimension > N, column offset; guard
columns checked).

  python tests/stress/fuzz_api.py --n 200 --seed 1 > gpurun_out/fuzz_api.log
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (the checker; this tool is test infrastructure)
from oracle import conv as oconv  # noqa: E402


def csr(rng, M, K, dens, kind="uniform"):
    if kind == "lognormal":
        m = rng.random((M, K)) < np.clip(dens * rng.lognormal(0.0, 1.0, size=(M, 1)), 0.0, 1.0)
    else:
        m = rng.random((M, K)) < dens
    rp = np.zeros(M + 1, np.int32)
    rp[1:] = np.cumsum(m.sum(1))
    ci = np.nonzero(m)[1].astype(np.int32)
    v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
    v[v == 0] = 0.01
    return rp, ci, v


def rel_err(Y, Yo, S):
    e = np.abs(Y.astype(np.float64) - Yo) / np.where(S > 0, S, 1.0)
    ok = np.isfinite(Y).all() and float(e.max(initial=0.0)) <= 1e-4 and np.all(Y[S == 0] == Yo[S == 0])
    return ok, float(e.max(initial=0.0))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_2101_07948_b200 as sdnn

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(args.seed)
    fails, counts, t0 = 0, {}, time.time()
    for case in range(args.n):
        mode = str(rng.choice(["conv", "conv", "host", "chain", "multi"]))
        counts[mode] = counts.get(mode, 0) + 1
        try:
            if mode == "conv":
                OC, IC = int(rng.integers(1, 300)), int(rng.integers(1, 200))
                FY, FX = (int(rng.choice([1, 3, 3, 3, 5])),) * 2 if rng.random() < 0.8 else (int(rng.choice([1, 3])), int(rng.choice([1, 3, 5])))
                pad, stride = int(rng.integers(0, 3)), int(rng.choice([1, 1, 2]))
                H, W, B = int(rng.integers(max(1, FY - 2 * pad), 40)), int(rng.integers(max(1, FX - 2 * pad), 40)), int(rng.integers(1, 9))
                dens = float(rng.choice([0.02, 0.05, 0.1, 0.2, 0.5]))
                rp, ci, v = csr(rng, OC, IC * FY * FX, dens)
                use_b, act = bool(rng.random() < 0.8), int(rng.random() < 0.7)
                b = (0.1 * rng.standard_normal(OC)).astype(np.float32) if use_b else None
                X = rng.standard_normal((IC, B, H, W)).astype(np.float32)
                tag = f"conv OC={OC} IC={IC} {FY}x{FX} pad={pad} s={stride} {H}x{W} B={B} d={dens} nnz={ci.size} bias={use_b} act={act}"
                h = sdnn.Handle.for_conv(rp, ci, v, OC, IC, FY, FX)
                Yo, S = oconv.conv2d(rp, ci, v, OC, IC, FY, FX, X, pad, stride, b, act)
                Xd = torch.from_numpy(X).to(dev)
                bd = None if b is None else torch.from_numpy(b).to(dev)
                msgs = []
                Y1 = h.conv2d(Xd, FY, FX, pad, stride, bd, act).cpu().numpy()
                ok, e = rel_err(Y1, Yo, S)
                if not ok:
                    msgs.append(f"PARITY {e:.3e}")
                if not np.array_equal(h.conv2d(Xd, FY, FX, pad, stride, bd, act).cpu().numpy(), Y1):
                    msgs.append("NONDETERMINISTIC")
                if rng.random() < 0.4:
                    t = h.conv2d_tune(Xd, FY, FX, pad, stride)
                    ok, e = rel_err(h.conv2d(Xd, FY, FX, pad, stride, bd, act).cpu().numpy(), Yo, S)
                    if not ok:
                        msgs.append(f"TUNED {t} {e:.3e}")
                h.close()
            elif mode == "host":
                M, K, N = int(rng.integers(1, 1500)), int(rng.integers(1, 1500)), int(rng.integers(1, 20000))
                dens = float(rng.choice([0.02, 0.1, 0.3]))
                rp, ci, v = csr(rng, M, K, dens, str(rng.choice(["uniform", "lognormal"])))
                b = (0.1 * rng.standard_normal(M)).astype(np.float32) if rng.random() < 0.8 else None
                act = int(rng.random() < 0.7)
                X = rng.standard_normal((K, N)).astype(np.float32)
                bc = int(rng.choice([0, 0, 128, 1000, 4096, 1 << 20]))
                tag = f"host M={M} K={K} N={N} d={dens} nnz={ci.size} block_cols={bc} bias={b is not None} act={act}"
                h = sdnn.Handle(rp, ci, v, M, K)
                Yo, S, _ = oracle.spmm_omp(rp, ci, v, M, K, X, b, act=act, want_scale=True)
                Y1 = h.spmm_host(X, b, act, block_cols=bc)
                msgs = []
                ok, e = rel_err(Y1, Yo, S)
                if not ok:
                    msgs.append(f"PARITY {e:.3e}")
                Yd = h.spmm(torch.from_numpy(X).to(dev), None if b is None else torch.from_numpy(b).to(dev), act).cpu().numpy()
                e2 = np.abs(Yd.astype(np.float64) - Y1) / np.where(S > 0, S, 1.0)  # block N may take another plan: tolerance
                if float(e2.max(initial=0.0)) > 2e-4:
                    msgs.append(f"HOST vs DEVICE {e2.max():.3e}")
                h.close()
            elif mode == "chain":
                L = int(rng.integers(2, 4))
                dims = [int(rng.integers(8, 900)) for _ in range(L + 1)]
                N = int(rng.choice([64, 128, 500, 1024, 2048]))
                layers, ref = [], []
                for i in range(L):
                    M, K = dims[i + 1], dims[i]
                    rp, ci, v = csr(rng, M, K, float(rng.choice([0.05, 0.1, 0.3])), str(rng.choice(["uniform", "lognormal"])))
                    b = (0.1 * rng.standard_normal(M)).astype(np.float32) if rng.random() < 0.8 else None
                    act = 1 if i < L - 1 else int(rng.random() < 0.5)
                    layers.append((rp, ci, v, M, K, b, act))
                tag = f"chain dims={dims} N={N}"
                X = rng.standard_normal((dims[0], N)).astype(np.float32)
                ch = sdnn.Chain(layers)
                Y1 = ch.forward(torch.from_numpy(X).to(dev)).cpu().numpy()
                # oracle: layer by layer in fp64-accumulate, feeding each layer the ORACLE's fp32 output; the
                # tolerance scale of the last layer plus the propagated input error (a few ulp of each layer)
                # forward error bound: T_l = u·S_l + |W_l|·T_(l-1) (ReLU is 1-Lipschitz): the per-element bound
                # relative to S does not compose across layers (a near-zero intermediate carries the previous
                # layer's absolute error), so the previous layer's tolerance is pushed through |W_l|
                cur, T = X, np.zeros_like(X)
                u = 1e-5
                for (rp, ci, v, M, K, b, act) in layers:
                    cur, S, _ = oracle.spmm_omp(rp, ci, v, M, K, cur, b, act=act, want_scale=True)
                    Tp, _, _ = oracle.spmm_omp(rp, ci, np.abs(v), M, K, T.astype(np.float32), None, act=0, want_scale=True)
                    T = u * S + Tp.astype(np.float64) * (1 + 1e-6)
                d = np.abs(Y1.astype(np.float64) - cur)
                bad = d > T
                msgs = [] if (np.isfinite(Y1).all() and not bad.any()) else [f"PARITY {int(bad.sum())} elements beyond the propagated bound, worst {float((d / np.where(T > 0, T, 1)).max()):.3e} x bound"]
                if not np.array_equal(ch.forward(torch.from_numpy(X).to(dev)).cpu().numpy(), Y1):
                    msgs.append("NONDETERMINISTIC")
            else:  # multi
                M, K = int(rng.integers(1, 1200)), int(rng.integers(1, 1200))
                N = int(rng.choice([4, 100, 128, 512, 1000, 2048, 4100]))
                nd, col0 = int(rng.integers(1, 5)), 4 * int(rng.integers(0, 40))
                ld = col0 + N + 4 * int(rng.integers(0, 40))
                rp, ci, v = csr(rng, M, K, float(rng.choice([0.02, 0.1, 0.3])))
                b = (0.1 * rng.standard_normal(M)).astype(np.float32)
                X = rng.standard_normal((K, N)).astype(np.float32)
                kern = str(rng.choice(["auto", "row", "tmem"]))
                tag = f"multi M={M} K={K} N={N} dsts={nd} ld={ld} col0={col0} kernel={kern}"
                h = sdnn.Handle(rp, ci, v, M, K, kernel=kern)
                Yo, S, _ = oracle.spmm_omp(rp, ci, v, M, K, X, b, act=1, want_scale=True)
                dsts = [torch.full((M, ld), float("nan"), dtype=torch.float32, device=dev) for _ in range(nd)]
                h.spmm_multi(torch.from_numpy(X).to(dev), [d.data_ptr() for d in dsts], ld, col0, torch.from_numpy(b).to(dev), 1)
                torch.cuda.synchronize()
                msgs = []
                for i, d in enumerate(dsts):
                    dn = d.cpu().numpy()
                    ok, e = rel_err(dn[:, col0:col0 + N], Yo, S)
                    if not ok:
                        msgs.append(f"dst {i} PARITY {e:.3e}")
                    if not (np.isnan(dn[:, :col0]).all() and np.isnan(dn[:, col0 + N:]).all()):
                        msgs.append(f"dst {i} wrote outside its columns")
                    if i and not np.array_equal(dn[:, col0:col0 + N], dsts[0].cpu().numpy()[:, col0:col0 + N]):
                        msgs.append(f"dst {i} != dst 0")
                h.close()
            status = "ok" if not msgs else "FAIL " + "; ".join(msgs)
        except Exception as e:  # noqa: BLE001
            status = f"FAIL exception {type(e).__name__}: {e}"
            tag = locals().get("tag", mode)
        if status != "ok":
            fails += 1
        print(f"case {case}: {tag} -> {status}", flush=True)
    print(f"# {args.n} cases, {fails} failed, modes {counts}, {time.time() - t0:.0f} s")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
