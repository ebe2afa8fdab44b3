"""Time one configuration with one kernel (CUDA events, mean of --iters launches after warm-up).
usage: python tools/time_cfg.py --config c5 --kernel tmem [--n N] [--iters 5]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SDNN_PKG_DIR"):  # A/B runs: another build of the package (tools/jobs/ab.sh)
    sys.path.insert(0, os.environ["SDNN_PKG_DIR"])

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--kernel", default="tmem")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--opts", default="", help="handle options, e.g. panel_rows=4,cta_panels=4")
    ap.add_argument("--shape", default="", help="MxK:sparsity, e.g. 4096x2048:0.9 (uniform mask; overrides --config)")
    a = ap.parse_args()
    if a.shape:
        mk, sp = a.shape.split(":")
        M, K = (int(v) for v in mk.split("x"))
        p = synth.make_problem(a.shape, M, K, a.n or 65536, float(sp))
        a.config = a.shape
    else:
        p = synth.config_problem(a.config)
    N = a.n or p.N
    X = torch.randn((p.K, N), device="cuda")
    b = torch.from_numpy(p.bias).cuda()
    Y = torch.empty((p.M, N), device="cuda")
    for k in a.kernel.split(","):
        opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opts.split(",") if kv}
        h = sdnn.Handle.from_problem(p, kernel=k, **opts)
        for _ in range(2):
            h.spmm(X, b, act=1, out=Y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            h.spmm(X, b, act=1, out=Y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        print(f"{a.config} N={N} {k:8s} {a.opts:24s} lib={sdnn.LIB_PATH.split('/')[-3]} dbg={os.environ.get('SDNN_DEBUG_TMEM', '0')} {ms:9.3f} ms "
              f"{2 * p.nnz * N / ms / 1e9:8.2f} TF", flush=True)
        h.close()


if __name__ == "__main__":
    main()
