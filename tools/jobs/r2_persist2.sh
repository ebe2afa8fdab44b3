# persistent TMEM-R CTAs vs one CTA per item after the round-2 epilogue / start-up changes (graph-timed configs + c5)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p2_build.log 2>&1
for i in 1 2; do
  timeout 300 python tools/pdl_ab.py --configs c2_3072x768,c2_768x3072,c3_256x128,c3_512x512,c3_1024x512,c4_2048x512_s80,c4_512x2048_s80,c4_2048x512_s95,c4_512x2048_s95 | sed 's/^/P0 /' >> gpurun_out/p2.log 2>&1
  SDNN_TMEM_PERSIST=1 timeout 300 python tools/pdl_ab.py --configs c2_3072x768,c2_768x3072,c3_256x128,c3_512x512,c3_1024x512,c4_2048x512_s80,c4_512x2048_s80,c4_2048x512_s95,c4_512x2048_s95 | sed 's/^/P1 /' >> gpurun_out/p2.log 2>&1
done
cat gpurun_out/p2.log
