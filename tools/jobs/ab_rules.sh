#!/bin/bash
# graph-timed A/B of the per-call rules: ab/old (before the narrow4 / split-K / tile rules) vs this tree.
mkdir -p gpurun_out; rm -f gpurun_out/ab_rules_*.jsonl
for v in old new; do
  if [ $v = old ]; then export SDNN_PKG_DIR=ab/old; else unset SDNN_PKG_DIR; fi
  timeout 900 python tools/sweep.py --sdnn-only --sizes 1024,2048,3072,4096 --sparsity 0.7,0.9,0.95 \
    --ns ${NS:-64,128,256,1024} > gpurun_out/ab_rules_$v.jsonl 2> gpurun_out/ab_rules_$v.err
done
