# TMEM plans with fewer rows per warp (more row blocks, slots partly empty): SDNN_TMEM_ROWS = 10 (default) / 9 / 8 / 7
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rows_build.log 2>&1
for R in 0; do
  timeout 300 python tools/pdl_ab.py --configs c2_3072x768,c2_768x3072,c3_256x128,c3_512x512,c3_1024x512,c4_2048x512_s80,c4_512x2048_s95 | sed "s/^/R$R /" >> gpurun_out/rows_ab.log 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-proxy --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^/R$R /" >> gpurun_out/rows_ab.log
done
cat gpurun_out/rows_ab.log | cut -c1-200
