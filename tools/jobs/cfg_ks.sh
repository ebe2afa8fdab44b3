#!/bin/bash
# BASELINE configs, graph-timed, with the row split-K forced (SDNN_SPLIT_K) vs the rules.
mkdir -p gpurun_out; rm -f gpurun_out/cfg_ks_*.jsonl
for ks in 0 2 4; do
  if [ $ks = 0 ]; then unset SDNN_SPLIT_K; else export SDNN_SPLIT_K=$ks; fi
  timeout 600 python tools/bench_configs.py --variants auto --graph > gpurun_out/cfg_ks_$ks.jsonl 2> gpurun_out/cfg_ks_$ks.err
done
