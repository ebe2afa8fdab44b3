for v in A B C; do
  for d in 0 5; do SDNN_DEBUG_TMEM=$d SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --config c5 --kernel tmem --n 65536 | sed "s/^/$v /"; done
done
