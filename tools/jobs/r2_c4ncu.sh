# ncu --set full of the TMEM-R kernel on c4 2048x512 at 95 % (warm L2), source-level
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c4ncu_build.log 2>&1
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:spmm_tmemr -s 2 -c 1 \
  -o gpurun_out/c4_95_full python tools/prof_one.py --config c4_2048x512_s95 --kernel auto --launches 4 > gpurun_out/c4ncu.log 2>&1
tail -3 gpurun_out/c4ncu.log
