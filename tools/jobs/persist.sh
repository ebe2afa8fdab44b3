timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py -m gpu -q -x -k "tmem or auto or multi or gather or config_parity or smoke" 2>&1 | tail -3
for r in 1 2; do for pe in 0 1; do
  SDNN_TMEM_PERSIST=$pe timeout 120 python tools/time_cfg.py --config c5 --kernel tmem,tmem8 --iters 5 | sed "s/^/P$pe /"
done; done
for c in c4_2048x512_s80 c4_512x2048_s95 c3_512x512 c3_1024x512 c2_3072x768; do for pe in 0 1; do
  SDNN_TMEM_PERSIST=$pe timeout 120 python tools/time_cfg.py --config $c --kernel auto --iters 20 | sed "s/^/P$pe /"
done; done
