#!/bin/bash
# conv tile grid: rules vs forced (pixels per lane, K slices) per geometry (SDNN_CONV_PX / _KS).
mkdir -p gpurun_out; rm -f gpurun_out/convgrid.log
for cfg in "0 0" "2 1" "2 2" "2 4" "2 8" "4 1" "4 2" "4 4" "4 8"; do
  set -- $cfg
  SDNN_CONV_PX=$1 SDNN_CONV_KS=$2 timeout 600 python - <<'PY' >> gpurun_out/convgrid.log 2>&1
import os, sys, torch
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
tag = f"px={os.environ['SDNN_CONV_PX']} ks={os.environ['SDNN_CONV_KS']}"
for C in (32, 64, 128, 256, 512):
    for hw in (7, 14, 28, 56):
        for sp in (0.9, 0.95):
            if C * C * hw * hw > 512 * 512 * 28 * 28: continue
            p = synth.make_conv_problem(f"cg{C}_{hw}_{sp}", C, C, hw, hw, 8, sp)
            h = sdnn.Handle.for_conv(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3)
            X = torch.from_numpy(p.x()).cuda(); b = torch.from_numpy(p.bias).cuda()
            Y = torch.empty((p.OC, p.B, p.Ho, p.Wo), device="cuda")
            for _ in range(3): h.conv2d(X, 3, 3, 1, 1, b, act=1, out=Y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(20): h.conv2d(X, 3, 3, 1, 1, b, act=1, out=Y)
            e1.record(); torch.cuda.synchronize()
            print(f"{tag} C={C} HW={hw} sp={sp} {e0.elapsed_time(e1) / 20 * 1e3:.2f}", flush=True)
            h.close()
PY
done
echo "exit=$?" >> gpurun_out/convgrid.log
