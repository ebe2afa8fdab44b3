# TMEM-R panel groups: G CTAs per (row block, N tile) item, forced via SDNN_TMEM_G
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1
for G in 1 2 3 6; do SDNN_TMEM_G=$G timeout 300 python tools/pdl_ab.py --configs c2_3072x768,c2_768x3072,c3_256x128,c3_512x512,c3_1024x512,c4_2048x512_s80,c4_512x2048_s80,c4_2048x512_s95,c4_512x2048_s95 | sed "s/^/G$G /" >> gpurun_out/g_ab.log 2>&1; done
SDNN_TMEM_G=3 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tmem or config or c5 or desk" > gpurun_out/g_pytest.log 2>&1
SDNN_TMEM_G=6 timeout 600 python -m pytest tests/test_gpu_jitter.py -m gpu -q -x > gpurun_out/g_pytest6.log 2>&1
cat gpurun_out/g_ab.log; tail -2 gpurun_out/g_pytest.log gpurun_out/g_pytest6.log
