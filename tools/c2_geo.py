"""c2 768² geometry sweep (graph-timed): panel rows × CTA panels × stage depth (SDNN_ROW_STAGES set by
the caller per process)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import paper_2101_07948_b200 as sdnn  # noqa: E402
import sdnn_synth as synth  # noqa: E402
from pdl_ab import graph_time  # noqa: E402
key = sys.argv[1] if len(sys.argv) > 1 else "c2_768x768"
p = synth.config_problem(key)
X = torch.from_numpy(p.x()).cuda(); b = torch.from_numpy(p.bias).cuda(); Y = torch.empty((p.M, p.N), device="cuda")
for rw in (2, 4, 8):
    for wc in (2, 3, 4, 6, 8, 12):
        try:
            h = sdnn.Handle.from_problem(p, kernel="row", panel_rows=rw, cta_panels=wc)
        except Exception as e:  # noqa: BLE001
            continue
        us = graph_time(lambda: h.spmm(X, b, act=1, out=Y), 5)
        inf = h.info()
        print(json.dumps({"cfg": key, "stages": os.environ.get("SDNN_ROW_STAGES", "auto"), "rw": rw, "wc": wc,
                          "rb": inf["num_row_blocks"], "pieces": inf["num_pieces"], "us": round(us, 2)}), flush=True)
