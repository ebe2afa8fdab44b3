#!/bin/bash
# V = 2 vs V = 4 row tiles on the small-N narrow / narrow4 calls (SDNN_ROW_V forces the choice).
mkdir -p gpurun_out
for v in 0 2 4; do
  SDNN_ROW_V=$v timeout 600 python - <<'PY' >> gpurun_out/rowv.log 2>&1
import os, sys, torch
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
def timer(h, X, Y):
    for _ in range(3): h.spmm(X, None, act=1, out=Y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): h.spmm(X, None, act=1, out=Y)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 20 * 1e3
v = os.environ.get("SDNN_ROW_V")
for S, K in ((1024, 1024), (2048, 2048), (3072, 3072), (4096, 4096), (768, 3072), (512, 4096), (3072, 768)):
    for sp in (0.7, 0.9, 0.95):
        p = synth.make_problem(f"rv{S}_{sp}", S, K, 128, sp)
        h = sdnn.Handle.from_problem(p)
        row = []
        for N in (64, 128, 256):
            X = torch.randn((K, N), device="cuda"); Y = torch.empty((S, N), device="cuda")
            row.append(f"N={N} {timer(h, X, Y):7.2f}")
        h.close()
        print(f"V={v} {S}x{K}:{sp} " + " ".join(row), flush=True)
PY
done
echo "exit=$?" >> gpurun_out/rowv.log
