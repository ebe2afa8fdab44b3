#!/bin/bash
mkdir -p gpurun_out
NS=64,128 bash tools/jobs/ab_rules.sh
timeout 900 python -m pytest tests -m gpu -x -q -k "narrow or tune or serial or split or small" > gpurun_out/ab2_pytest.log 2>&1
echo "pytest exit=$?" >> gpurun_out/ab2_pytest.log
