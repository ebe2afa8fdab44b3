#!/bin/bash
# host rules (narrow4, TMEM split-K FLOP floor): affected GPU tests, auto-vs-tuned grid, full sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "narrow or tune or serial or split or guard or small" > gpurun_out/r4_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/r4_pytest.log
bash tools/jobs/tune_grid.sh
cp gpurun_out/tune_grid.log gpurun_out/r4_tune_grid.log
timeout 1200 python tools/sweep.py --out gpurun_out/sweep8.jsonl > gpurun_out/sweep8.log 2>&1
echo "sweep exit=$?" >> gpurun_out/sweep8.log
