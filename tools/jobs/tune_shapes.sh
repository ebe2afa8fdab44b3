python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
for M, K, sp in [(4096, 4096, 0.9), (2048, 2048, 0.9), (1024, 1024, 0.7), (768, 3072, 0.9), (512, 4096, 0.95), (3072, 768, 0.9)]:
    p = synth.make_problem(f"ts{M}_{K}", M, K, 128, sp)
    h = sdnn.Handle.from_problem(p)
    for N in (128, 256, 512, 1024, 2048):
        X = torch.randn((K, N), device="cuda"); Y = torch.empty((M, N), device="cuda")
        def t():
            for _ in range(3): h.spmm(X, None, act=1, out=Y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(20): h.spmm(X, None, act=1, out=Y)
            e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 20 * 1e3
        a = t(); r = h.tune(X); tt = t()
        print(f"{M}x{K}:{sp} N={N:5d} auto {a:8.2f} us tuned {tt:8.2f} us {r['path']}/{r['split_k']}", flush=True)
PY
