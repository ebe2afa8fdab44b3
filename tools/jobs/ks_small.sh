#!/bin/bash
# graph-timed: default rules vs forced row split-K (SDNN_SPLIT_K) on small shapes with 4-16 K chunks.
mkdir -p gpurun_out; rm -f gpurun_out/ks_small_*.jsonl
for ks in 0 2 4 8; do
  if [ $ks = 0 ]; then unset SDNN_SPLIT_K; else export SDNN_SPLIT_K=$ks; fi
  timeout 600 python tools/sweep.py --sdnn-only --sizes 256,512,768,1024 --sparsity 0.7,0.9,0.95 \
    --ns 64,128,256,512 > gpurun_out/ks_small_$ks.jsonl 2> gpurun_out/ks_small_$ks.err
done
