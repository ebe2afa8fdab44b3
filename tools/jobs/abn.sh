# A/B/n timing of several builds of the package in one GPU session (ab/<name> each; VARIANTS="A B C")
for round in 1 2; do for v in ${VARIANTS:-A B}; do
  SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --config ${CFG:-c5} --kernel ${KERN:-tmem} --iters ${ITERS:-5} | sed "s/^/$v /"
done; done
