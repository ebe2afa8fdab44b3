"""Randomised stress of sdnn_spmm against the oracle on a GPU (a bug hunt, wider than the hypothesis
test in tests/test_gpu_parity.py: M, K up to 5000, N up to 8192, heavy-tailed rows, every plan kind the
per-call rules can reach — TMEM-R / second TMEM plan / persistent / split-K / row / narrow / narrow4 /
V = 2 — with guard zones around Y, repeat-run determinism, sdnn_tune and a serialize round trip).

  python tests/stress/fuzz.py --n 300 --seed 1 > gpurun_out/fuzz.log
Prints one line per case and a summary; exit code 1 if any case failed.
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
import sdnn_synth as synth  # noqa: E402


def draw_dim(rng, hi, anchors):
    """A dimension near one of the geometry boundaries, or log-uniform."""
    if rng.random() < 0.5:
        a = int(rng.choice(anchors)) * int(rng.integers(1, 6))
        return int(np.clip(a + int(rng.integers(-3, 4)), 1, hi))
    return int(np.clip(np.exp(rng.uniform(0, np.log(hi))), 1, hi))


def draw_mask(rng, M, K, dens, kind):
    if kind == "blocks4":
        m = np.repeat(rng.random((M, (K + 3) // 4)) < dens, 4, axis=1)[:, :K]
    elif kind == "lognormal":
        row_d = np.clip(dens * rng.lognormal(0.0, 1.0, size=(M, 1)), 0.0, 1.0)
        m = rng.random((M, K)) < row_d
    elif kind == "heavy":  # a few dense rows among sparse ones
        m = rng.random((M, K)) < dens
        for r in rng.choice(M, size=min(M, 3), replace=False):
            m[r] = rng.random(K) < 0.9
    else:
        m = rng.random((M, K)) < dens
    return m


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-dim", type=int, default=5000)
    ap.add_argument("--max-n", type=int, default=8192)
    ap.add_argument("--max-gflop", type=float, default=12.0)
    ap.add_argument("--big", action="store_true", help="M, K in [400, max-dim], N a multiple of 4 in [512, max-n]")
    ap.add_argument("--wide-n", action="store_true", help="short K (1-12 chunks), many N tiles: persistent / wave-fill rules")
    args = ap.parse_args()

    import torch
    import paper_2101_07948_b200 as sdnn

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(args.seed)
    fails = 0
    kinds = {}
    t_start = time.time()
    for case in range(args.n):
        M = draw_dim(rng, args.max_dim, [240, 96, 64, 32, 16, 4])
        K = draw_dim(rng, args.max_dim, [64, 128, 8])
        if rng.random() < 0.6:
            N = int(np.clip(128 * int(rng.integers(1, args.max_n // 128 + 1)) + int(rng.choice([0, 0, 0, 4, -4, 1, 64])), 1, args.max_n))
        else:
            N = int(np.clip(np.exp(rng.uniform(0, np.log(args.max_n))), 1, args.max_n))
        if args.big:
            M, K = int(rng.integers(400, args.max_dim + 1)), int(rng.integers(400, args.max_dim + 1))
            N = int(rng.integers(128, args.max_n // 4 + 1)) * 4 if rng.random() < 0.5 else 128 * int(rng.integers(4, args.max_n // 128 + 1))
        if args.wide_n:
            M = int(rng.integers(100, args.max_dim + 1))
            K = int(np.clip(64 * int(rng.integers(1, 13)) + int(rng.choice([0, 0, -1, 1, -30])), 1, None))
            N = 128 * int(rng.integers(8, max(9, args.max_n // 128 + 1))) + int(rng.choice([0, 0, 0, 4, 64, 1]))
        dens = float(rng.choice([0.0, 0.005, 0.02, 0.05, 0.1, 0.2, 0.5, 1.0], p=[.03, .1, .15, .2, .25, .15, .09, .03]))
        while 2.0 * dens * M * K * N > args.max_gflop * 1e9 and N > 128:
            N //= 2
        mk = str(rng.choice(["uniform", "blocks4", "lognormal", "heavy"]))
        m = draw_mask(rng, M, K, dens, mk)
        rp = np.zeros(M + 1, np.int32)
        rp[1:] = np.cumsum(m.sum(1))
        ci = np.nonzero(m)[1].astype(np.int32)
        v = (0.05 * rng.standard_normal(ci.size)).astype(np.float32)
        v[v == 0] = 0.01
        use_bias, act = bool(rng.random() < 0.8), int(rng.random() < 0.7)
        b = (0.1 * rng.standard_normal(M)).astype(np.float32) if use_bias else None
        X = rng.standard_normal((K, N)).astype(np.float32)
        kernel = str(rng.choice(["auto", "auto", "auto", "auto", "row", "tmem", "tmemp", "tmem8", "group"]))
        opts = dict(kernel=kernel, permute=bool(rng.random() < 0.9))
        if kernel == "group":
            opts["group_sb"] = int(rng.choice([0, 1, 2, 4]))
        if kernel == "row" and rng.random() < 0.5:
            opts.update(panel_rows=int(rng.choice([4, 8])), cta_panels=int(rng.choice([1, 2, 4, 8, 16])),
                        k_chunk=int(rng.choice([0, 8, 32, 64, 96])))
        if rng.random() < 0.15:
            opts["split_k"] = False
        if rng.random() < 0.15:
            opts["split_rows"] = False
        if rng.random() < 0.1:
            opts["permuted_output"] = True
        off_x, off_y = (int(rng.integers(0, 4)) if rng.random() < 0.15 else 0 for _ in range(2))  # misalignment in floats
        tag = f"case {case}: M={M} K={K} N={N} d={dens} {mk} nnz={ci.size} {opts} bias={use_bias} act={act} offx={off_x} offy={off_y}"
        try:
            try:
                h = sdnn.Handle(rp, ci, v, M, K, **opts)
            except sdnn.SdnnError as pe:
                # an explicit K chunk whose two stages do not fit shared memory: documented SDNN_ERR_UNSUPPORTED
                if pe.status == 3 and opts.get("k_chunk"):
                    print(f"{tag} -> skipped (explicit k_chunk does not fit)", flush=True)
                    continue
                raise
            Yo, S, _ = oracle.spmm_omp(rp, ci, v, M, K, X, b, act=act, want_scale=True)
            if opts.get("permuted_output"):
                perm = h.permutation()
                Yo, S = Yo[perm], S[perm]
                bq = None if b is None else b[perm]
            else:
                bq = b
            G = 64  # guard floats on both sides of Y
            xbuf = torch.empty(K * N + 8, dtype=torch.float32, device=dev)
            Xd = xbuf[off_x:off_x + K * N].view(K, N)
            Xd.copy_(torch.from_numpy(X))
            ybuf = torch.full((M * N + 2 * G + 8,), float("nan"), dtype=torch.float32, device=dev)
            Yd = ybuf[G + off_y:G + off_y + M * N].view(M, N)
            bd = None if bq is None else torch.from_numpy(np.ascontiguousarray(bq)).to(dev)
            kid = h.kernel_for(N, Xd.data_ptr(), Yd.data_ptr())
            kinds[kid] = kinds.get(kid, 0) + 1
            h.spmm(Xd, bd, act=act, out=Yd)
            torch.cuda.synchronize()
            Y1 = Yd.cpu().numpy()
            guards = torch.cat([ybuf[:G + off_y], ybuf[G + off_y + M * N:]])
            msgs = []
            if not bool(torch.isnan(guards).all()):
                msgs.append("GUARD overwritten")
            err = np.abs(Y1.astype(np.float64) - Yo) / np.where(S > 0, S, 1.0)
            if not (np.isfinite(Y1).all() and float(err.max(initial=0.0)) <= 1e-4 and np.all(Y1[S == 0] == Yo[S == 0])):
                msgs.append(f"PARITY max err/S {err.max(initial=0.0):.3e} finite={np.isfinite(Y1).all()}")
            ybuf.fill_(float("nan"))
            h.spmm(Xd, bd, act=act, out=Yd)
            if not np.array_equal(Yd.cpu().numpy(), Y1):
                msgs.append("NONDETERMINISTIC repeat")
            if kernel not in ("codegen",) and rng.random() < 0.3:  # serialize round trip: bitwise
                h2 = sdnn.Handle.deserialize(h.serialize())
                ybuf.fill_(float("nan"))
                h2.spmm(Xd, bd, act=act, out=Yd)
                if not np.array_equal(Yd.cpu().numpy(), Y1):
                    msgs.append("DESERIALIZED handle differs")
                h2.close()
            if off_x == 0 and off_y == 0 and N % 4 == 0 and rng.random() < 0.4:  # tuned path (needs N % 4 == 0, aligned): parity again
                try:
                    t = h.tune(Xd, out=Yd)
                except sdnn.SdnnError as te:
                    if te.status != 3:  # SDNN_ERR_UNSUPPORTED: this handle kind is not tuned
                        raise
                    t = None
                if t is not None:
                    ybuf.fill_(float("nan"))
                    h.spmm(Xd, bd, act=act, out=Yd)
                    Y3 = Yd.cpu().numpy()
                    e3 = np.abs(Y3.astype(np.float64) - Yo) / np.where(S > 0, S, 1.0)
                    guards = torch.cat([ybuf[:G + off_y], ybuf[G + off_y + M * N:]])
                    if not (np.isfinite(Y3).all() and float(e3.max(initial=0.0)) <= 1e-4 and bool(torch.isnan(guards).all())):
                        msgs.append(f"TUNED path {t} parity {e3.max(initial=0.0):.3e}")
            h.close()
            status = "ok" if not msgs else "FAIL " + "; ".join(msgs)
        except Exception as e:  # noqa: BLE001
            status = f"FAIL exception {type(e).__name__}: {e}"
        if status != "ok":
            fails += 1
        print(f"{tag} -> {status}", flush=True)
    print(f"# {args.n} cases, {fails} failed, kernel ids {dict(sorted(kinds.items()))}, {time.time() - t_start:.0f} s")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
