"""Sparse convolution suite (IC/OC 32-256, images 7/14/28/56, 3×3, pad 1,
90 / 95 %): per-launch time in a CUDA graph of sdnn_conv2d against cuDNN dense fp32 convolution
(torch conv2d on the densified filters, TF32 off) — the paper compares against oneDNN dense (3.0-6.3×
geomean on CPU).  Batch --batch (CNHW activations for sdnn, NCHW for cuDNN).
usage: python tools/conv_bench.py [--batch 8] [--out FILE]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SDNN_PKG_DIR"):  # A/B runs: another build of the package
    sys.path.insert(0, os.environ["SDNN_PKG_DIR"])

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402
from tools.sweep import graph_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    ap.add_argument("--cta-panels", type=int, default=0, help="row-plan warps per CTA (0 = auto)")
    ap.add_argument("--k-chunk", type=int, default=-1, help="row-plan K chunk (-1 = Handle.for_conv's choice, 0 = auto)")
    ap.add_argument("--sizes", default="32,64,128,256")
    ap.add_argument("--images", default="7,14,28,56")
    a = ap.parse_args()
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    out = open(a.out, "w") if a.out else None
    sp_all = {0.9: [], 0.95: []}
    for ch in (int(v) for v in a.sizes.split(",")):
        for hw in (int(v) for v in a.images.split(",")):
            for sp in (0.9, 0.95):
                p = synth.make_conv_problem(f"cb{ch}_{hw}_{sp}", ch, ch, hw, hw, a.batch, sp)
                h = sdnn.Handle.for_conv(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3, cta_panels=a.cta_panels,
                                         **({"k_chunk": a.k_chunk} if a.k_chunk >= 0 else {}))
                X = torch.from_numpy(p.x()).cuda()
                b = torch.from_numpy(p.bias).cuda()
                Y = torch.empty((p.OC, p.B, p.Ho, p.Wo), device="cuda")
                t_s = graph_time(lambda: h.conv2d(X, 3, 3, 1, 1, b, act=1, out=Y), a.reps)
                Wd = torch.zeros((p.OC, p.K))
                rows = torch.repeat_interleave(torch.arange(p.OC), torch.from_numpy(p.row_ptr[1:] - p.row_ptr[:-1]).long())
                Wd[rows, torch.from_numpy(p.col_idx).long()] = torch.from_numpy(p.vals)
                Wd = Wd.reshape(p.OC, p.IC, 3, 3).cuda()
                Xn = X.permute(1, 0, 2, 3).contiguous()
                Yn = torch.empty((p.B, p.OC, p.Ho, p.Wo), device="cuda")

                def dense():
                    torch.clamp_min(torch.nn.functional.conv2d(Xn, Wd, b, padding=1), 0.0, out=Yn)

                t_d = graph_time(dense, a.reps)
                flops = 2 * p.nnz * p.B * p.Ho * p.Wo
                rec = {"C": ch, "HW": hw, "sparsity": sp, "B": p.B, "sdnn_us": round(t_s, 2),
                       "cudnn_dense_us": round(t_d, 2), "speedup_vs_dense": round(t_d / t_s, 2),
                       "sdnn_tflops": round(flops / t_s / 1e6, 3)}
                sp_all[sp].append(t_d / t_s)
                print(json.dumps(rec), flush=True)
                if out:
                    out.write(json.dumps(rec) + "\n")
                h.close()
    summ = {f"geomean_speedup_vs_cudnn_dense_{int(s * 100)}": round(statistics.geometric_mean(v), 3)
            for s, v in sp_all.items()}
    print(json.dumps(summ), flush=True)
    if out:
        out.write(json.dumps(summ) + "\n")
        out.close()


if __name__ == "__main__":
    main()
