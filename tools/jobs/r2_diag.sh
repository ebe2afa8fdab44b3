# TMEM-R time decomposition: product vs no-consumer-loop (DIAG 3) vs no-fill (DIAG 4) vs no TMA (runtime)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/diag_build.log 2>&1
timeout 300 python tools/tmemr_diag.py product >> gpurun_out/diag.log 2>&1
SDNN_DEBUG_TMEM=1 timeout 300 python tools/tmemr_diag.py product >> gpurun_out/diag.log 2>&1
for d in 3 4; do
  SDNN_NVCC_FLAGS="-DSDNN_DIAG=$d" python paper_2101_07948_b200/build.py --force >> gpurun_out/diag_build.log 2>&1
  timeout 300 python tools/tmemr_diag.py diag$d >> gpurun_out/diag.log 2>&1
  SDNN_DEBUG_TMEM=1 timeout 300 python tools/tmemr_diag.py diag$d >> gpurun_out/diag.log 2>&1
done
python paper_2101_07948_b200/build.py --force >> gpurun_out/diag_build.log 2>&1
cat gpurun_out/diag.log
