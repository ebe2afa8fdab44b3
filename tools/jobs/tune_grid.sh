#!/bin/bash
# auto rules vs sdnn_tune over square shapes × sparsity × small N, then narrow geometries at M = 4096.
mkdir -p gpurun_out
timeout 1200 python - > gpurun_out/tune_grid.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
def timer(h, X, Y):
    for _ in range(3): h.spmm(X, None, act=1, out=Y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): h.spmm(X, None, act=1, out=Y)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 20 * 1e3
for S in (1024, 2048, 4096):
    for sp in (0.7, 0.8, 0.9, 0.95):
        p = synth.make_problem(f"tg{S}_{sp}", S, S, 128, sp)
        h = sdnn.Handle.from_problem(p)
        for N in (128, 256, 512, 1024):
            X = torch.randn((S, N), device="cuda"); Y = torch.empty((S, N), device="cuda")
            k = h.kernel_for(N, X.data_ptr(), Y.data_ptr())
            a = timer(h, X, Y); r = h.tune(X); tt = timer(h, X, Y)
            print(f"{S}x{S}:{sp} N={N:5d} auto k={k} {a:8.2f} us tuned {tt:8.2f} us {r['path']}/{r['split_k']} gain {a/tt:5.2f}", flush=True)
        h.close()
print("--- narrow geometries")
for S in (4096, 3072, 2048):
    for sp in (0.7, 0.8, 0.9, 0.95):
        p = synth.make_problem(f"ng{S}_{sp}", S, S, 128, sp)
        for N in (128, 256):
            X = torch.randn((S, N), device="cuda"); Y = torch.empty((S, N), device="cuda")
            h = sdnn.Handle.from_problem(p); a = timer(h, X, Y); h.close()
            row = [f"auto {a:7.2f}"]
            for cp in (4, 8, 16):
                h = sdnn.Handle.from_problem(p, kernel="row", panel_rows=4, cta_panels=cp)
                row.append(f"4x{cp} {timer(h, X, Y):7.2f}"); h.close()
            print(f"{S}x{S}:{sp} N={N:4d} " + " ".join(row), flush=True)
PY
echo "exit=$?" >> gpurun_out/tune_grid.log
