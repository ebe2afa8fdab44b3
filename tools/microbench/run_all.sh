#!/bin/bash
# microbenchmarks on the box (B3b); output -> gpurun_out/microbench.log
cd "$(dirname "$0")"
python gen_bigcode.py  # bigcode*.inc for peaks.cu (generated, not committed)
mkdir -p ../../gpurun_out
{
echo "== host"; nproc; grep -m1 "model name" /proc/cpuinfo; free -g | head -2; python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
echo "== peaks"; timeout 120 ./peaks
echo "== probe small O0 (code fits I-cache)"; timeout 120 ./run_probe probe_small.cubin 836 4
echo "== probe small O3"; timeout 120 ./run_probe probe_small_O3.cubin 836 4
echo "== probe big O0 (13192 fma/iter, ~300KB code per variant)"; timeout 300 ./run_probe probe_big.cubin 13192 4
} > ../../gpurun_out/microbench.log 2>&1
