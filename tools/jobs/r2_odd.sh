timeout 200 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 --n 65536
timeout 200 python tools/time_cfg.py --config c5 --kernel tmem --iters 5
for cfg in c2_3072x768 c3_512x512 c3_1024x512 c4_2048x512_s80 c4_512x2048_s95; do timeout 200 python tools/time_cfg.py --config $cfg --kernel tmem --iters 30; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_serialize.py -q -x -k "tmem" 2>&1 | tail -3
