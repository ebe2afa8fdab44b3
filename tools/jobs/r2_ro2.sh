# runs-only consumer with the next run's metadata read during this run's loads
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/ro2_build.log 2>&1
for i in 1 2; do timeout 300 python tools/pdl_ab.py --configs c4_2048x512_s80,c4_512x2048_s80,c4_2048x512_s95,c4_512x2048_s95 >> gpurun_out/ro2_ab.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_guards.py -m gpu -q -x > gpurun_out/ro2_pytest.log 2>&1
tail -1 gpurun_out/ro2_build.log; grep -v chain gpurun_out/ro2_ab.log; tail -2 gpurun_out/ro2_pytest.log
