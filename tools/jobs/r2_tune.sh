# auto rules vs sdnn_tune after the TMEM-R kernel: BASELINE configs and the round-1 tuned-shape grid
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
def timeit(h, X, Y, b):
    for _ in range(3): h.spmm(X, b, act=1, out=Y)
    s_ = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s_):
        for _ in range(20): h.spmm(X, b, act=1, out=Y)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20 * 1e3
cases = [(k, synth.config_problem(k)) for k in synth.CONFIGS if k != "c5"]
for M, K, sp in [(4096, 4096, 0.9), (2048, 2048, 0.9), (1024, 1024, 0.7), (768, 3072, 0.9), (512, 4096, 0.95), (3072, 768, 0.9)]:
    for N in (128, 512, 2048):
        cases.append((f"{M}x{K}:{sp}:N{N}", synth.make_problem(f"ts{M}_{K}", M, K, N, sp)))
for name, p in cases:
    h = sdnn.Handle.from_problem(p)
    X = torch.randn((p.K, p.N), device="cuda"); Y = torch.empty((p.M, p.N), device="cuda")
    b = torch.from_numpy(p.bias).cuda() if p.bias is not None else None
    k0 = h.kernel_for(p.N, X.data_ptr(), Y.data_ptr())
    a = timeit(h, X, Y, b); r = h.tune(X, out=Y); t = timeit(h, X, Y, b)
    print(f"{name:28s} N={p.N:6d} auto {a:9.2f} us (kernel {k0})  tuned {t:9.2f} us {r['path']}/{r['split_k']}  gain {a / t:5.2f}x", flush=True)
PY
