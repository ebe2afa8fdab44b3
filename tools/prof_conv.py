"""Launch one sparse conv (target for ncu).  usage: python tools/prof_conv.py C HW B sparsity"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402

C, HW, B, sp = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
p = synth.make_conv_problem("pc", C, C, HW, HW, B, sp)
h = sdnn.Handle.for_conv(p.row_ptr, p.col_idx, p.vals, p.OC, p.IC, 3, 3)
print(h.info())
X = torch.from_numpy(p.x()).cuda()
b = torch.from_numpy(p.bias).cuda()
for _ in range(2):
    h.conv2d(X, 3, 3, 1, 1, b, act=1)
torch.cuda.synchronize()
print("ok")
