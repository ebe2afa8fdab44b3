# kernel 6 (Algorithm 1 row pairs) vs kernel 4: parity subset, then timings
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_serialize.py -q -x -k "tmemp" 2>&1 | tail -4
for cfg in c2_3072x768 c2_768x3072 c3_512x512 c3_1024x512 c4_2048x512_s80 c4_2048x512_s95; do
  timeout 200 python tools/time_cfg.py --config $cfg --kernel tmem,tmemp --iters 30
done
timeout 200 python tools/time_cfg.py --config c5 --kernel tmem,tmemp --iters 5 --n 65536
timeout 200 python tools/time_cfg.py --config c5 --kernel tmem,tmemp --iters 5 --n 65536 --opts permute=0
