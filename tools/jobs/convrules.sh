#!/bin/bash
# conv split-K rule change: conv GPU tests, rules-only grid, conv bench vs cuDNN.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "conv" > gpurun_out/cr_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/cr_pytest.log
sed -i 's/^for cfg in .*/for cfg in "0 0"; do/' tools/jobs/convgrid.sh
bash tools/jobs/convgrid.sh
cp gpurun_out/convgrid.log gpurun_out/cr_grid.log
timeout 900 python tools/conv_bench.py --out gpurun_out/cr_bench.jsonl > gpurun_out/cr_bench.log 2>&1
echo "bench exit=$?" >> gpurun_out/cr_bench.log
