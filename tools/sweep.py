"""Paper-style sweep (the shape of the paper's E1 grid) on one B200:
square W of size 256..2048 (and 4096), sparsity 70..95 % (uniform mask), N in {128, 512, 2048}, bias + ReLU.

Per point, per-launch time (CUDA graph of --reps launches, replayed; inputs L2-resident for the small
sizes, as in the paper's per-layer timing) of
  * sdnn      — this library, auto kernel choice (sdnn_spmm through the C ABI);
  * cusparse  — torch.sparse CSR @ dense (cuSPARSE SpMM, fp32), + bias + ReLU as torch ops;
  * dense     — cuBLAS SGEMM on the densified W (TF32 off), + bias + ReLU: the dense break-even
                (the paper's "when does sparse pay").
Library calls are context baselines only (the product path never calls them).  Each point also
checks sdnn against the cuSPARSE result (max |diff| / (|W||X| + |b|)).

usage: python tools/sweep.py [--sizes 256,512,1024,2048] [--sparsity 0.7,0.8,0.9,0.95] [--ns 128,512,2048]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SDNN_PKG_DIR"):  # A/B runs: another build of the package
    sys.path.insert(0, os.environ["SDNN_PKG_DIR"])

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (3 * reps)  # µs per launch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="256,512,1024,2048,4096")
    ap.add_argument("--sparsity", default="0.7,0.8,0.9,0.95")
    ap.add_argument("--ns", default="128,512,2048")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    ap.add_argument("--sdnn-only", action="store_true", help="skip the library baselines (A/B of builds)")
    a = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    out = open(a.out, "w") if a.out else None
    for size in (int(v) for v in a.sizes.split(",")):
        for sp in (float(v) for v in a.sparsity.split(",")):
            p = synth.make_problem(f"sweep{size}_{sp}", size, size, 128, sp)
            h = sdnn.Handle.from_problem(p)
            Wd = torch.zeros((p.M, p.K), dtype=torch.float32)
            rows = np.repeat(np.arange(p.M), np.diff(p.row_ptr))
            Wd[torch.from_numpy(rows), torch.from_numpy(p.col_idx.astype(np.int64))] = torch.from_numpy(p.vals)
            Wd = Wd.cuda()
            Wsp = torch.sparse_csr_tensor(torch.from_numpy(p.row_ptr.astype(np.int64)),
                                          torch.from_numpy(p.col_idx.astype(np.int64)),
                                          torch.from_numpy(p.vals), size=(p.M, p.K)).cuda()
            b = torch.from_numpy(p.bias).cuda()
            for N in (int(v) for v in a.ns.split(",")):
                X = torch.randn((p.K, N), device="cuda")
                Y = torch.empty((p.M, N), device="cuda")
                t_sdnn = graph_time(lambda: h.spmm(X, b, act=1, out=Y), a.reps)
                kid = h.kernel_for(N, X.data_ptr(), Y.data_ptr())
                Ys = torch.empty_like(Y)

                def cusp():
                    torch.clamp_min((Wsp @ X) + b[:, None], 0.0, out=Ys)

                def dense():
                    torch.clamp_min(torch.addmm(b[:, None], Wd, X), 0.0, out=Ys)

                if a.sdnn_only:
                    print(json.dumps({"M": p.M, "sparsity": sp, "N": N, "kernel": kid, "sdnn_us": round(t_sdnn, 2),
                                      "lib": sdnn.LIB_PATH}), flush=True)
                    continue
                try:
                    t_cusp = graph_time(cusp, a.reps)
                except Exception as e:  # capture of the sparse op not supported: eager timing
                    print(f"cusparse graph capture failed ({e}); eager", file=sys.stderr)
                    for _ in range(3):
                        cusp()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.reps):
                        cusp()
                    e1.record()
                    torch.cuda.synchronize()
                    t_cusp = e0.elapsed_time(e1) * 1e3 / a.reps
                cusp()
                torch.cuda.synchronize()
                h.spmm(X, b, act=1, out=Y)
                scale = torch.abs(Wd) @ torch.abs(X) + torch.abs(b)[:, None]
                err = float((torch.abs(Y - Ys) / torch.clamp(scale, min=1e-30)).max())
                t_dense = graph_time(dense, a.reps)
                flops = 2 * p.nnz * N
                rec = {"M": p.M, "K": p.K, "sparsity": sp, "nnz": p.nnz, "N": N, "kernel": kid,
                       "sdnn_us": round(t_sdnn, 2), "cusparse_us": round(t_cusp, 2), "dense_us": round(t_dense, 2),
                       "sdnn_tflops": round(flops / t_sdnn / 1e6, 3),
                       "speedup_vs_cusparse": round(t_cusp / t_sdnn, 2), "speedup_vs_dense": round(t_dense / t_sdnn, 2),
                       "max_err_vs_cusparse_over_scale": err}
                print(json.dumps(rec), flush=True)
                if out:
                    out.write(json.dumps(rec) + "\n")
                del X, Y, Ys
            h.close()
    if out:
        out.close()


if __name__ == "__main__":
    main()
