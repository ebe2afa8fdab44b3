"""Launch one configuration a few times (target for ncu).  usage:
python tools/prof_one.py --config c5 --kernel tmem --n 32768 --launches 2"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--kernel", default="tmem")
    ap.add_argument("--n", type=int, default=0, help="override N (columns), 0 = the config's")
    ap.add_argument("--launches", type=int, default=2)
    a = ap.parse_args()
    p = synth.config_problem(a.config)
    N = a.n or p.N
    h = sdnn.Handle.from_problem(p, kernel=a.kernel)
    X = torch.randn((p.K, N), device="cuda")
    b = torch.from_numpy(p.bias).cuda()
    Y = torch.empty((p.M, N), device="cuda")
    for _ in range(a.launches):
        h.spmm(X, b, act=1, out=Y)
    torch.cuda.synchronize()
    print("ok", h.info())


if __name__ == "__main__":
    main()
