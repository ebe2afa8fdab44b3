# round-2 per-config ncu counters and the E1 sweep vs cuSPARSE / cuBLAS
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cnt_build.log 2>&1
rm -rf gpurun_out/cfgncu
bash tools/jobs/ncu_configs.sh
python tools/cfg_counters.py gpurun_out/cfgncu > gpurun_out/cfgncu/summary.jsonl 2> gpurun_out/cfgncu/summary.err
timeout 1500 python tools/sweep.py --out gpurun_out/r2s2_sweep.jsonl > gpurun_out/r2s2_sweep.log 2>&1
wc -l gpurun_out/cfgncu/summary.jsonl; tail -3 gpurun_out/r2s2_sweep.log
