"""c2 768² (pruneBERT attention-output shape, log-normal rows, N = 1024) under every plan / geometry
knob, graph-timed (20 back-to-back launches): which limit sets its ~20 µs.

usage: [SDNN_SPLIT_K=n] [SDNN_ROW_V=2|4] [SDNN_ROW_STAGES=n] python tools/c2_probe2.py [--config c2_768x768]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402
from pdl_ab import graph_time  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_768x768")
ap.add_argument("--variants", default="all")
args = ap.parse_args()
p = synth.config_problem(args.config)
X = torch.from_numpy(p.x()).cuda()
b = torch.from_numpy(p.bias).cuda()
Y = torch.empty((p.M, p.N), device="cuda")
env = {k: v for k, v in os.environ.items() if k.startswith("SDNN_")}
V = [dict(), dict(split_rows=False), dict(kernel="tmem"), dict(kernel="row", panel_rows=4, cta_panels=4),
     dict(kernel="row", panel_rows=4, cta_panels=8), dict(kernel="row", panel_rows=8, cta_panels=16),
     dict(kernel="row", panel_rows=4, cta_panels=2), dict(kernel="row", k_chunk=32),
     dict(kernel="row", k_chunk=32, panel_rows=4, cta_panels=4)]
ref = None
for opts in V:
    try:
        h = sdnn.Handle.from_problem(p, **opts)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"opts": opts, "error": str(e)[:120]}), flush=True)
        continue
    us = graph_time(lambda: h.spmm(X, b, act=1, out=Y), 5)
    if ref is None:
        ref = Y.clone()
    inf = h.info()
    err = float((Y - ref).abs().max())
    print(json.dumps({"env": env, "opts": opts, "us": round(us, 2), "kernel": h.kernel_for(p.N, X.data_ptr(), Y.data_ptr()),
                      "rb": inf.get("num_row_blocks"), "split_rows": inf.get("num_split_rows"),
                      "pieces": inf.get("num_pieces"), "kc": inf.get("k_chunk"), "max_abs_diff_vs_first": err}), flush=True)
h = sdnn.Handle.from_problem(p)
t = h.tune(X, out=Y)
print(json.dumps({"env": env, "tune": t}), flush=True)
