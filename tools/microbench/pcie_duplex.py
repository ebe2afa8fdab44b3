"""PCIe ceiling for the host entry point (sdnn_spmm_host, bench.py's e2e): pinned-host copies of
--gib GiB H2D alone, D2H alone, and both at once on two streams (the pipelined e2e overlaps them).
usage: python tools/microbench/pcie_duplex.py [--gib 1] [--reps 3]"""
import argparse

import torch


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n = int(a.gib * (1 << 30)) // 4
    hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
    dx = torch.empty(n, dtype=torch.float32, device="cuda")
    dy = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    b = n * 4

    def h2d():
        dx.copy_(hx, non_blocking=True)

    def d2h():
        hy.copy_(dy, non_blocking=True)

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            dx.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            hy.copy_(dy, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t1, t2, t3 = timed(h2d, a.reps), timed(d2h, a.reps), timed(both, a.reps)
    print(f"H2D alone {b / t1 / 1e9:6.1f} GB/s; D2H alone {b / t2 / 1e9:6.1f} GB/s; "
          f"both at once {2 * b / t3 / 1e9:6.1f} GB/s combined ({b / t3 / 1e9:5.1f} per direction)")
    c5 = 4294983680 + 4294967296  # bench.py e2e bytes per step (X + bias in, Y out)
    print(f"c5 e2e copy floor at the concurrent rate: {c5 / (2 * b / t3) * 1e3:6.1f} ms "
          f"(device kernel 51.1 ms overlaps it)")


if __name__ == "__main__":
    main()
