#!/bin/bash
# narrow4 plan + TMEM split-K rule: GPU tests of the affected paths, then auto vs tuned grid.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "narrow or tune or serial or split or guard or small" > gpurun_out/n4_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/n4_pytest.log
bash tools/jobs/tune_grid.sh
cp gpurun_out/tune_grid.log gpurun_out/n4_tune_grid.log
