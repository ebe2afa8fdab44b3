"""Per-config kernel timing (SURVEY §8(d) timing protocol): for each BASELINE config and kernel
variant, median of `--iters` launches bracketed by CUDA events, L2 flushed before each launch
(memset of a 2×L2 scratch buffer outside the events).  Prints one JSON line per (config, variant)
with effective GFLOP/s, algorithmic GB/s and the fraction of the fp32 / HBM roofline.

Also (--graph) the warm per-launch time: a CUDA graph of 50 back-to-back launches, replayed, time / 50
(the SURVEY §8(d) "warm" protocol; small configs then stay L2-resident and launch overhead is amortised).

usage: python tools/bench_configs.py [--configs c1,c2_768x768,...] [--variants auto,row,tmem,tmem8,group2] [--graph]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SDNN_PKG_DIR"):  # A/B runs: another build of the package
    sys.path.insert(0, os.environ["SDNN_PKG_DIR"])

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(k for k in synth.CONFIGS if k != "c5"))
    ap.add_argument("--variants", default="auto,row,group1,group2,group4")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warm", action="store_true", help="no L2 flush (L2-resident timing)")
    ap.add_argument("--graph", action="store_true", help="also time a CUDA graph of 50 launches")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    props = torch.cuda.get_device_properties(dev)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    fp32_peak = props.multi_processor_count * 128 * 2 * float(peaks.get("sm_max_mhz", 1965)) * 1e6
    hbm_peak = float(peaks.get("hbm_gbs", 6556.2)) * 1e9
    flush = torch.empty(2 * 126 * 2**20 // 4 + 1024, dtype=torch.float32, device=dev)
    for key in args.configs.split(","):
        p = synth.config_problem(key)
        X = torch.from_numpy(p.x()).to(dev)
        b = torch.from_numpy(p.bias).to(dev)
        Y = torch.empty((p.M, p.N), device=dev)
        flops = 2.0 * p.nnz * p.N
        alg_bytes = p.nnz * 8 + (p.K + p.M) * p.N * 4
        for var in args.variants.split(","):
            kw = dict(kernel="group", group_sb=int(var[-1])) if var.startswith("group") else dict(kernel=var)
            h = sdnn.Handle.from_problem(p, **kw)
            info = h.info()
            ts = []
            for i in range(args.iters + 3):
                if not args.warm:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                h.spmm(X, b, act=1, out=Y)
                e1.record()
                torch.cuda.synchronize()
                if i >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e-3)
            t = statistics.median(ts)
            graph_us = None
            if args.graph:
                s_ = torch.cuda.Stream()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s_):
                    for _ in range(50):
                        h.spmm(X, b, act=1, out=Y)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                graph_us = e0.elapsed_time(e1) * 1e3 / 50
                del g
            kid = h.kernel_for(p.N, X.data_ptr(), Y.data_ptr())
            print(json.dumps({"config": key, "variant": var, "kernel": info["kernel"], "launched": kid, "sb": info["group_sb"],
                              "M": p.M, "K": p.K, "N": p.N, "nnz": p.nnz, "us": round(t * 1e6, 2),
                              "gflops": round(flops / t / 1e9, 1), "gbs": round(alg_bytes / t / 1e9, 1),
                              "fp32_frac": round(flops / t / fp32_peak, 4), "hbm_frac": round(alg_bytes / t / hbm_peak, 4),
                              "roof_frac": round(max(flops / fp32_peak, alg_bytes / hbm_peak) / t, 4),
                              "l2": "warm" if args.warm else "flushed",
                              **({} if graph_us is None else {
                                  "graph_us": round(graph_us, 2), "graph_gflops": round(flops / graph_us / 1e3, 1),
                                  "graph_roof_frac": round(max(flops / fp32_peak, alg_bytes / hbm_peak) / (graph_us * 1e-6), 4)})}),
                  flush=True)
            h.close()


if __name__ == "__main__":
    main()
