"""sdnn_spmm_host (host buffers, H2D + kernel + D2H pipelined) on c5 for several column-block widths.
usage: python tools/e2e_blocks.py [--n 262144] [--blocks 0,4096,16384,65536]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SDNN_PKG_DIR"):  # A/B runs: another build of the package
    sys.path.insert(0, os.environ["SDNN_PKG_DIR"])

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--blocks", default="0,4096,16384,32768,65536")
    ap.add_argument("--kernel", default="auto")
    a = ap.parse_args()
    p = synth.config_problem("c5")
    N = a.n
    h = sdnn.Handle.from_problem(p, kernel=a.kernel)
    Xh = torch.randn((p.K, N)).pin_memory()
    Yh = torch.empty((p.M, N)).pin_memory()
    for bc in (int(x) for x in a.blocks.split(",")):
        h.spmm_host_ptr(Xh.data_ptr(), N, p.bias.ctypes.data, 1, Yh.data_ptr(), bc)
        t0 = time.perf_counter()
        for _ in range(3):
            h.spmm_host_ptr(Xh.data_ptr(), N, p.bias.ctypes.data, 1, Yh.data_ptr(), bc)
        dt = (time.perf_counter() - t0) / 3
        gb = (p.K + p.M) * N * 4 / 1e9
        print(f"block_cols={bc:6d}: {dt * 1e3:8.1f} ms  {2 * p.nnz * N / dt / 1e12:6.2f} TF  PCIe {gb / dt:6.1f} GB/s (H2D+D2H)",
              flush=True)
    # raw copy speeds for context
    Xd = torch.empty((p.K, N), device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter(); Xd.copy_(Xh, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    Yh.copy_(Xd[:p.M], non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"contiguous H2D {p.K * N * 4 / (t1 - t0) / 1e9:.1f} GB/s, D2H {p.M * N * 4 / (t2 - t1) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
