#!/bin/bash
# for_conv default of 8 panels per CTA: conv GPU tests and the graph-timed conv suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv" > gpurun_out/cc2_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/cc2_pytest.log
timeout 900 python tools/conv_bench.py --out gpurun_out/cc2_bench.jsonl > gpurun_out/cc2_bench.log 2>&1
