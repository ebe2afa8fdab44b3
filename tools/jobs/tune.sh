timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tune or split or narrow or auto_takes or bitwise or host" 2>&1 | tail -3
python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
for key, N in [("c2_768x3072", 1024), ("c2_768x768", 1024), ("c3_1024x512", 6272), ("c4_512x2048_s80", 12544), ("c1", 128)]:
    p = synth.config_problem(key)
    h = sdnn.Handle.from_problem(p)
    X = torch.randn((p.K, N), device="cuda"); Y = torch.empty((p.M, N), device="cuda"); b = torch.from_numpy(p.bias).cuda()
    def t():
        for _ in range(3): h.spmm(X, b, act=1, out=Y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(20): h.spmm(X, b, act=1, out=Y)
        e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 20 * 1e3
    a = t(); r = h.tune(X); tt = t()
    print(f"{key:18s} auto {a:8.2f} us   tuned {tt:8.2f} us   {r}", flush=True)
PY
