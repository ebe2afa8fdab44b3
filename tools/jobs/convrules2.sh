#!/bin/bash
# conv split-K rule, graph-timed: conv GPU tests and the conv suite vs cuDNN.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv" > gpurun_out/cr2_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/cr2_pytest.log
timeout 900 python tools/conv_bench.py --out gpurun_out/cr2_bench.jsonl > gpurun_out/cr2_bench.log 2>&1
echo "bench exit=$?" >> gpurun_out/cr2_bench.log
