"""Chained FFN pair: BERT-FFN shapes of c2 (768 → 3072 → 768, 90 %, log-normal rows,
ReLU between), per forward in a CUDA graph: the Chain (permutation carried across layers, no
un-permute, reused intermediate) against two independent sdnn_spmm calls (each un-permuting).
usage: python tools/chain_bench.py [--ns 1024,8192,32768]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402
from tools.sweep import graph_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="1024,8192,32768")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    w1, w2 = synth.config_problem("c2_3072x768"), synth.config_problem("c2_768x3072")
    chain = sdnn.Chain([(w1.row_ptr, w1.col_idx, w1.vals, w1.M, w1.K, w1.bias, 1),
                        (w2.row_ptr, w2.col_idx, w2.vals, w2.M, w2.K, w2.bias, 1)])
    h1, h2 = sdnn.Handle.from_problem(w1), sdnn.Handle.from_problem(w2)
    b1, b2 = torch.from_numpy(w1.bias).cuda(), torch.from_numpy(w2.bias).cuda()
    for N in (int(v) for v in a.ns.split(",")):
        X = torch.randn((w1.K, N), device="cuda")
        Y = torch.empty((w2.M, N), device="cuda")
        Y1 = torch.empty((w1.M, N), device="cuda")
        chain.forward(X, out=Y)
        t_chain = graph_time(lambda: chain.forward(X, out=Y), a.reps)

        def plain():
            h1.spmm(X, b1, act=1, out=Y1)
            h2.spmm(Y1, b2, act=1, out=Y)

        t_plain = graph_time(plain, a.reps)
        flops = 2 * (w1.nnz + w2.nnz) * N
        print(json.dumps({"N": N, "chain_us": round(t_chain, 2), "two_calls_us": round(t_plain, 2),
                          "chain_tflops": round(flops / t_chain / 1e6, 3), "speedup": round(t_plain / t_chain, 3),
                          "kernels": [h1.kernel_for(N), h2.kernel_for(N)]}), flush=True)


if __name__ == "__main__":
    main()
