#!/bin/bash
# conv: CTA height (panels per CTA) on the mid sizes, graph-timed (tools/conv_bench.py).
mkdir -p gpurun_out; rm -f gpurun_out/conv_cta_*.jsonl
for cp in 0 2 4 8 16; do
  timeout 600 python tools/conv_bench.py --cta-panels $cp --sizes 64,128,256 --images 7,14,28,56 \
    --out gpurun_out/conv_cta_$cp.jsonl > gpurun_out/conv_cta_$cp.log 2>&1
done
