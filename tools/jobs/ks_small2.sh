#!/bin/bash
# relaxed row split-K rule: full GPU suite, then graph-timed rules on the small shapes and the sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ks2_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/ks2_pytest.log
timeout 600 python tools/sweep.py --sdnn-only --sizes 256,512,768,1024 --sparsity 0.7,0.9,0.95 \
    --ns 64,128,256,512 > gpurun_out/ks_small_new.jsonl 2> gpurun_out/ks_small_new.err
timeout 1200 python tools/sweep.py --out gpurun_out/sweep10.jsonl > gpurun_out/sweep10.log 2>&1
