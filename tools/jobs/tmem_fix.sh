#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tf_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/tf_pytest.log
bash tools/jobs/tune_shapes.sh > gpurun_out/tune_shapes_fix.log 2>&1
