# ncu --set full of the c2 768² row-kernel launch (warm L2: --cache-control none), source-level
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2ncu_build.log 2>&1
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_tma_kernel -s 2 -c 1 \
  -o gpurun_out/c2_row_full python tools/prof_one.py --config c2_768x768 --kernel auto --launches 4 > gpurun_out/c2ncu.log 2>&1
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_tma_kernel -s 2 -c 1 \
  -o gpurun_out/c1_row_full python tools/prof_one.py --config c1 --kernel auto --launches 4 >> gpurun_out/c2ncu.log 2>&1
tail -5 gpurun_out/c2ncu.log
