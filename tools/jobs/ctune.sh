timeout 600 python -m pytest tests/test_gpu_conv.py -m gpu -q 2>&1 | tail -2
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
for C in (64, 128, 256):
    for hw in (7, 14, 28, 56):
        for sp in (0.9,):
            p = synth.make_conv_problem(f"cb{C}_{hw}_{sp}", C, C, hw, hw, 8, sp)
            h = sdnn.Handle.for_conv(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3)
            X = torch.from_numpy(p.x()).cuda(); b = torch.from_numpy(p.bias).cuda()
            Y = torch.empty((p.OC, p.B, p.Ho, p.Wo), device="cuda")
            def t():
                for _ in range(3): h.conv2d(X, 3, 3, 1, 1, b, act=1, out=Y)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(); e0.record()
                for _ in range(20): h.conv2d(X, 3, 3, 1, 1, b, act=1, out=Y)
                e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 20 * 1e3
            a = t(); r = h.conv2d_tune(X); tt = t()
            print(f"C={C:3d} HW={hw:2d} sp={sp} rules {a:8.2f} us tuned {tt:8.2f} us {r}", flush=True)
PY
