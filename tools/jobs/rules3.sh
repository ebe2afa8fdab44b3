timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split or tune or narrow" 2>&1 | tail -2
bash tools/jobs/tune_shapes.sh > gpurun_out/tune_shapes3.log 2>&1
