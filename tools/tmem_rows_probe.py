"""TMEM plans at fewer rows per warp (kernel 4, panel_rows_max = r: more row blocks) on small calls,
each tuned over TMEM split-K (sdnn_tune on a kernel-4 handle: slices 1/2/4/8), against the auto
handle's choice.  usage: python tools/tmem_rows_probe.py [configs]"""
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

keys = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2_768x768", "c3_256x128", "c2_768x3072", "c3_512x512"]
for key in keys:
    p = synth.config_problem(key)
    X = torch.from_numpy(p.x()).cuda()
    b = torch.from_numpy(p.bias).cuda()
    Y = torch.empty((p.M, p.N), device="cuda")
    h = sdnn.Handle.from_problem(p)
    print(json.dumps({"config": key, "plan": "auto", "us": round(graph_time(lambda: h.spmm(X, b, act=1, out=Y), 3), 2)}),
          flush=True)
    for r in (10, 8, 6, 4, 3, 2):
        try:
            ht = sdnn.Handle.from_problem(p, kernel="tmem", panel_rows=r)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"config": key, "rows": r, "error": str(e)[:80]}), flush=True)
            continue
        t = ht.tune(X, out=Y)
        us = graph_time(lambda: ht.spmm(X, b, act=1, out=Y), 3)
        print(json.dumps({"config": key, "rows": r, "rb": ht.info()["num_row_blocks"], "tuned": t, "us": round(us, 2)}),
              flush=True)
