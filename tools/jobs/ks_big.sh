#!/bin/bash
# graph-timed: rules vs forced row split-K on 2048-4096², N 64-256 (long K ranges, 1-2-wave grids).
mkdir -p gpurun_out; rm -f gpurun_out/ks_big_*.jsonl
for ks in 0 2 4; do
  if [ $ks = 0 ]; then unset SDNN_SPLIT_K; else export SDNN_SPLIT_K=$ks; fi
  timeout 600 python tools/sweep.py --sdnn-only --sizes 2048,3072,4096 --sparsity 0.7,0.9,0.95 \
    --ns 64,128,256 > gpurun_out/ks_big_$ks.jsonl 2> gpurun_out/ks_big_$ks.err
done
