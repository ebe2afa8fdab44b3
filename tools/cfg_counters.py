"""Summarise the per-config ncu counter captures (tools/jobs/ncu_configs.sh → <dir>/<config>.csv) into
one JSON line per (config, kernel launch): time, DRAM bytes against the algorithmic bytes, L2 bytes,
FMA-pipe activity, IPC, tcgen05.ld count, shared-memory wavefronts / conflicts.

usage: python tools/cfg_counters.py <dir> > <dir>/summary.jsonl
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import sdnn_synth as synth  # noqa: E402

NAMES = {
    "gpu__time_duration.sum": ("time_us", 1e-3),
    "dram__bytes_read.sum": ("dram_rd_MB", 1e-6),
    "dram__bytes_write.sum": ("dram_wr_MB", 1e-6),
    "lts__t_bytes.sum": ("l2_MB", 1e-6),
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": ("fma_pipe_pct", 1.0),
    "sm__inst_executed.avg.per_cycle_active": ("ipc", 1.0),
    "smsp__sass_inst_executed_op_tmem_ldt.sum": ("tmem_ld", 1.0),
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": ("smem_wavefronts", 1.0),
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": ("smem_conflicts", 1.0),
    "launch__grid_size": ("grid", 1.0),
    "launch__registers_per_thread": ("regs", 1.0),
}


def main(d):
    for f in sorted(os.listdir(d)):
        if not f.endswith(".csv"):
            continue
        key = f[:-4]
        cfg = "c5" if key.startswith("c5") else key
        p = synth.config_problem(cfg, N=4)
        N = 65536 if cfg == "c5" else synth.CONFIGS[cfg][2]
        alg_mb = (p.nnz * 8 + (p.K + p.M) * N * 4) * 1e-6
        launches = {}
        with open(os.path.join(d, f)) as fh:
            rows = [r for r in csv.reader(fh)]
        hdr = None
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if not hdr or len(r) != len(hdr):
                continue
            rec = dict(zip(hdr, r))
            ent = launches.setdefault(rec["ID"], {"config": key, "kernel": rec["Kernel Name"].split("(")[0]})
            name = NAMES.get(rec["Metric Name"])
            if name:
                try:
                    ent[name[0]] = round(float(rec["Metric Value"].replace(",", "")) * name[1], 3)
                except ValueError:
                    pass
        for ent in launches.values():
            ent["alg_MB"] = round(alg_mb, 2)
            print(json.dumps(ent))


if __name__ == "__main__":
    main(sys.argv[1])
