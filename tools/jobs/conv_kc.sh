timeout 600 python -m pytest tests/test_gpu_conv.py -m gpu -q 2>&1 | tail -2
for kc in 0 72; do timeout 900 python tools/conv_bench.py --k-chunk $kc --out gpurun_out/conv_kc$kc.jsonl > gpurun_out/conv_kc$kc.log 2>&1; done
