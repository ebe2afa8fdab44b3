#!/bin/bash
# Small-N / low-sparsity probe (tools/small_n_probe.py) on one B200.
mkdir -p gpurun_out
timeout 900 python tools/small_n_probe.py > gpurun_out/smalln.log 2>&1
echo "exit=$?" >> gpurun_out/smalln.log
