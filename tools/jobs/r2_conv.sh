# conv explicit form (im2col + TMEM-R): parity, then the suite with the form on (default rule) / off
timeout 900 python -m pytest tests/test_gpu_conv.py -q -x 2>&1 | tail -3
SDNN_CONV_IM2COL=0 timeout 900 python tools/conv_bench.py --out gpurun_out/r2_conv_patch.jsonl > /dev/null 2>&1
timeout 900 python tools/conv_bench.py --out gpurun_out/r2_conv_rule.jsonl > /dev/null 2>&1
SDNN_CONV_IM2COL=1 timeout 900 python tools/conv_bench.py --out gpurun_out/r2_conv_explicit.jsonl > /dev/null 2>&1
tail -1 gpurun_out/r2_conv_patch.jsonl gpurun_out/r2_conv_rule.jsonl gpurun_out/r2_conv_explicit.jsonl
