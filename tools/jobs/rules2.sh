timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_conv.py -m gpu -q -x -k "split or tune or conv or narrow" 2>&1 | tail -2
timeout 900 python tools/conv_bench.py --out gpurun_out/conv_bench9.jsonl > gpurun_out/conv_bench9.log 2>&1
bash tools/jobs/tune_shapes.sh > gpurun_out/tune_shapes2.log 2>&1
