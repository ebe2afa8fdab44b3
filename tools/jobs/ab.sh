# A/B timing of two builds of the package in one GPU session (ab/A = baseline, ab/B = candidate)
for round in 1 2; do for v in A B; do
  SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --config ${CFG:-c5} --kernel ${KERN:-tmem} --iters ${ITERS:-5} | sed "s/^/$v /"
done; done
