import sys, os, torch
sys.path.insert(0, ".")
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
p = synth.config_problem("c2_768x768")
X = torch.from_numpy(p.x()).cuda(); b = torch.from_numpy(p.bias).cuda(); Y = torch.empty((p.M, p.N), device="cuda")
def gt(h):
    for _ in range(3): h.spmm(X, b, act=1, out=Y)
    s_ = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s_):
        for _ in range(20): h.spmm(X, b, act=1, out=Y)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20 * 1e3
for opts in [dict(), dict(split_rows=False), dict(kernel="row", split_rows=False), dict(kernel="row", split_rows=False, panel_rows=4),
             dict(kernel="row", panel_rows=4, cta_panels=4), dict(kernel="row", panel_rows=4, cta_panels=2, split_rows=False)]:
    h = sdnn.Handle.from_problem(p, **opts)
    print(os.environ.get("SDNN_SPLIT_K", "-"), opts, h.kernel_for(p.N, X.data_ptr(), Y.data_ptr()), round(gt(h), 2), "us", flush=True)
