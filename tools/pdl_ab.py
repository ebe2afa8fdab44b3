"""Graph-timed per-launch time of the BASELINE configs c1-c4 (auto kernel choice), and of a dependent
two-layer chain (pruneBERT FFN: 3072×768 then 768×3072, the second layer reading the first's Y), for
an A/B of programmatic dependent launch: run once with SDNN_PDL=0 and once without.  Every graph's
output is checked bitwise against an eager (synchronised) run of the same calls.

usage: [SDNN_PDL=0] python tools/pdl_ab.py [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402


def graph_time(fn, reps, launches=20):
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s_)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s_):
        for _ in range(launches):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / launches * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--configs", default=",".join(k for k in synth.CONFIGS if k != "c5"))
    args = ap.parse_args()
    pdl = os.environ.get("SDNN_PDL", "1")
    dev = torch.device("cuda", 0)
    for key in args.configs.split(","):
        p = synth.config_problem(key)
        X = torch.from_numpy(p.x()).to(dev)
        b = torch.from_numpy(p.bias).to(dev)
        h = sdnn.Handle.from_problem(p)
        Y0 = h.spmm(X, b, act=1)
        torch.cuda.synchronize()
        Y = torch.full_like(Y0, float("nan"))
        us = graph_time(lambda: h.spmm(X, b, act=1, out=Y), args.reps)
        ok = bool(torch.equal(Y, Y0))
        print(json.dumps({"pdl": pdl, "local_pieces": os.environ.get("SDNN_LOCAL_PIECES", "1"), "config": key, "kernel": h.kernel_for(p.N, X.data_ptr(), Y.data_ptr()),
                          "us": round(us, 2), "bitwise_eq_eager": ok}), flush=True)
    # dependent chain: Y1 = relu(W1 X + b1) (3072×768), Y2 = relu(W2 Y1 + b2) (768×3072)
    p1 = synth.config_problem("c2_3072x768")
    p2 = synth.config_problem("c2_768x3072")
    h1, h2 = sdnn.Handle.from_problem(p1), sdnn.Handle.from_problem(p2)
    X = torch.from_numpy(p1.x()).to(dev)
    b1, b2 = torch.from_numpy(p1.bias).to(dev), torch.from_numpy(p2.bias).to(dev)
    Y1e = h1.spmm(X, b1, act=1)
    torch.cuda.synchronize()
    Y2e = h2.spmm(Y1e, b2, act=1)
    torch.cuda.synchronize()
    Y1 = torch.full_like(Y1e, float("nan"))
    Y2 = torch.full_like(Y2e, float("nan"))

    def chain():
        h1.spmm(X, b1, act=1, out=Y1)
        h2.spmm(Y1, b2, act=1, out=Y2)
        Y1.fill_(float("nan"))  # a third kernel writes Y1 after layer 2 read it (WAR across PDL launches)

    us = graph_time(chain, args.reps, launches=10)  # Y2 as the graph's last layer 2 wrote it
    print(json.dumps({"pdl": pdl, "local_pieces": os.environ.get("SDNN_LOCAL_PIECES", "1"), "config": "ffn_chain_3072x768_768x3072", "us_per_pair": round(us, 2),
                      "bitwise_eq_eager": bool(torch.equal(Y2, Y2e))}), flush=True)


if __name__ == "__main__":
    main()
