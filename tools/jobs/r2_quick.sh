# quick c5 timing + tmem parity subset
timeout 300 python tools/time_cfg.py --config c5 --kernel tmem --n 65536 --iters 5 2>&1
timeout 300 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 2>&1
timeout 300 python tools/time_cfg.py --config c4_2048x512_s80 --kernel tmem --iters 20 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tmem" 2>&1 | tail -3
