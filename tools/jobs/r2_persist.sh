# persistent TMEM-R CTAs for short K: parity (ab_parity through the default build = auto rules) + A/B by env
SDNN_TMEM_PERSIST=1 timeout 300 python tools/ab_parity.py 2>&1 | tail -14
for cfg in c2_3072x768 c3_256x128 c3_512x512 c3_1024x512 c4_2048x512_s80 c4_512x2048_s80 c4_2048x512_s95 c4_512x2048_s95; do
  for pe in 0 1; do SDNN_TMEM_PERSIST=$pe timeout 100 python tools/time_cfg.py --config $cfg --kernel tmem --iters 30 | sed "s/^/persist=$pe /"; done
done
for pe in 0 1; do SDNN_TMEM_PERSIST=$pe timeout 100 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 | sed "s/^/persist=$pe /"; done
