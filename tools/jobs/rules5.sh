#!/bin/bash
# row-tile V rule (N <= 64 → V = 2; split-K calls → V = 4): affected GPU tests, V grid, sweep.
mkdir -p gpurun_out
rm -f gpurun_out/rowv.log
timeout 900 python -m pytest tests -m gpu -x -q -k "narrow or tune or serial or split or guard or small or ragged or chain or c1 or c2" > gpurun_out/r5_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/r5_pytest.log
bash tools/jobs/rowv.sh
cp gpurun_out/rowv.log gpurun_out/r5_rowv.log
timeout 1200 python tools/sweep.py --out gpurun_out/sweep9.jsonl > gpurun_out/sweep9.log 2>&1
echo "sweep exit=$?" >> gpurun_out/sweep9.log
