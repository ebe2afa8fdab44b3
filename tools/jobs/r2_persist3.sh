# automatic persistent TMEM-R CTAs (short K, many items): configs, jitter / persistence tests, parity
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p3_build.log 2>&1
timeout 300 python tools/pdl_ab.py > gpurun_out/p3_ab.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_jitter.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/p3_pytest.log 2>&1
tail -1 gpurun_out/p3_build.log; cat gpurun_out/p3_ab.log; tail -3 gpurun_out/p3_pytest.log
