for r in 1 2 3; do for f in 1 2; do SDNN_TMEM_FILL=$f timeout 200 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 | sed "s/^/fill=$f /"; done; done
for c in c4_2048x512_s80 c4_512x2048_s80 c4_2048x512_s95 c3_1024x512 c3_512x512 c2_3072x768; do for f in 1 2; do SDNN_TMEM_FILL=$f timeout 120 python tools/time_cfg.py --config $c --kernel tmem --iters 30 | sed "s/^/fill=$f /"; done; done
SDNN_TMEM_FILL=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tmem and not tmem8" 2>&1 | tail -2
