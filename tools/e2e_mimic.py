import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, numpy as np
import paper_2101_07948_b200 as sdnn, sdnn_synth as synth
p = synth.config_problem("c5"); N = p.N
h = sdnn.Handle.from_problem(p)
Xh = torch.randn((p.K, N)).pin_memory(); Yh = torch.empty((p.M, N)).pin_memory()
def e2e(tag):
    h.spmm_host_ptr(Xh.data_ptr(), N, p.bias.ctypes.data, 1, Yh.data_ptr())
    t0 = time.perf_counter()
    for _ in range(3): h.spmm_host_ptr(Xh.data_ptr(), N, p.bias.ctypes.data, 1, Yh.data_ptr())
    print(tag, f"{(time.perf_counter() - t0) / 3 * 1e3:.1f} ms", flush=True)
e2e("fresh")
X = Xh.cuda(); Y = torch.empty((p.M, N), device="cuda"); b = torch.from_numpy(p.bias).cuda()
e2e("after device alloc")
for _ in range(5): h.spmm(X, b, act=1, out=Y)
torch.cuda.synchronize()
e2e("after device launches")
del X, Y
torch.cuda.empty_cache()
e2e("after free")
