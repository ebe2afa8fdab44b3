"""TMEM-R time decomposition (graph-timed): the product build against diagnostic builds
(SDNN_DIAG=3: consumers skip their entry streams; 4: issuers skip the tcgen05.cp fill) and the
runtime switch SDNN_DEBUG_TMEM=1 (no X TMA loads).  Results of the diagnostic runs are wrong by
design; only their times are read.  usage: [SDNN_DEBUG_TMEM=1] python tools/tmemr_diag.py <label>"""
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

label = sys.argv[1] if len(sys.argv) > 1 else "product"
for key, N in (("c4_2048x512_s95", None), ("c4_2048x512_s80", None), ("c3_512x512", None), ("c2_3072x768", None),
               ("c5", 16384)):
    p = synth.config_problem(key, N=N) if N else synth.config_problem(key)
    X = torch.from_numpy(p.x_cols(0, p.N) if key == "c5" else p.x()).cuda()
    b = torch.from_numpy(p.bias).cuda()
    Y = torch.empty((p.M, p.N), device="cuda")
    h = sdnn.Handle.from_problem(p, kernel="tmem")
    us = graph_time(lambda: h.spmm(X, b, act=1, out=Y), 3, launches=10)
    print(json.dumps({"build": label, "debug_tmem": os.environ.get("SDNN_DEBUG_TMEM", "0"), "config": key, "N": p.N,
                      "us": round(us, 2)}), flush=True)
