"""Concurrency stress: several host threads share one prepared handle, each on its own CUDA stream, and
call sdnn_spmm / sdnn_spmm_host with different N (row plan, split-K workspace, TMEM-R, TMEM split-K,
persistent) in a loop; every result must be bitwise the single-threaded one (ctypes drops the GIL, so
the calls really overlap).

  python tests/stress/fuzz_threads.py --threads 4 --iters 60 > gpurun_out/fuzz_threads.log
"""
from __future__ import annotations

import argparse
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import sdnn_synth as synth  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=4)
    ap.add_argument("--iters", type=int, default=60)
    args = ap.parse_args()
    import torch
    import paper_2101_07948_b200 as sdnn

    dev = torch.device("cuda", 0)
    fails = 0
    shapes = [("c2_768x3072", [128, 256, 1024, 2048]), ("c2_768x768", [64, 128, 1024]), ("c4_2048x512_s95", [512, 12544]),
              ("c3_512x512", [100, 6272])]
    for key, Ns in shapes:
        p = synth.config_problem(key, N=max(Ns))
        h = sdnn.Handle.from_problem(p)
        Xfull = torch.from_numpy(p.x()).to(dev)
        bias = torch.from_numpy(p.bias).to(dev)
        Xs = {n: Xfull[:, :n].contiguous() for n in Ns}
        ref = {n: h.spmm(Xs[n], bias, act=1).clone() for n in Ns}
        Xh = {n: Xs[n].cpu().numpy() for n in Ns[:2]}
        torch.cuda.synchronize()
        errors = []

        def worker(t):
            try:
                st = torch.cuda.Stream(device=dev)
                rng = np.random.default_rng(t)
                with torch.cuda.stream(st):
                    for it in range(args.iters):
                        n = int(rng.choice(Ns))
                        if n in Xh and rng.random() < 0.15:
                            Y = torch.from_numpy(h.spmm_host(Xh[n], p.bias, 1)).to(dev)
                        else:
                            Y = h.spmm(Xs[n], bias, act=1, stream=st)
                        st.synchronize()
                        if not torch.equal(Y, ref[n]):
                            errors.append(f"thread {t} iter {it} N={n}: result differs from the single-threaded one")
            except Exception as e:  # noqa: BLE001
                errors.append(f"thread {t}: {type(e).__name__}: {e}")

        ths = [threading.Thread(target=worker, args=(t,)) for t in range(args.threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        print(f"{key} Ns={Ns}: {args.threads} threads x {args.iters} calls -> {'ok' if not errors else 'FAIL'}", flush=True)
        for e in errors[:5]:
            print("   ", e)
        fails += len(errors)
        h.close()
    print(f"# {fails} failures")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
