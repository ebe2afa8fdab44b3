for round in 1 2; do for v in A B C; do
  SDNN_PKG_DIR=ab/$v timeout 200 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 --n 65536 | sed "s/^/$v /"
done; done
