# end-of-round evidence refresh: per-config ncu counters and the E1 sweep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rf_build.log 2>&1
rm -rf gpurun_out/cfgncu
bash tools/jobs/ncu_configs.sh
python tools/cfg_counters.py gpurun_out/cfgncu > gpurun_out/cfgncu/summary.jsonl 2> gpurun_out/cfgncu/summary.err
timeout 1500 python tools/sweep.py --out gpurun_out/r2s2_sweep2.jsonl > gpurun_out/r2s2_sweep2.log 2>&1
wc -l gpurun_out/cfgncu/summary.jsonl; tail -1 gpurun_out/r2s2_sweep2.log
