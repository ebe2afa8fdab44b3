for d in 0 5 2; do SDNN_DEBUG_TMEM=$d timeout 120 python tools/time_cfg.py --config c5 --kernel tmem,tmem8 --n 65536; done
