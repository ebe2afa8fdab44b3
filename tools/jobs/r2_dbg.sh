for d in 0 4 8 16 24; do SDNN_DEBUG_TMEM=$d timeout 200 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 --n 65536; done
