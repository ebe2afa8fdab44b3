# runs-only TMEM-R consumer (block-clustered masks): c4 configs graph-timed, parity / jitter / pdl tests
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/ro_build.log 2>&1
for i in 1 2; do timeout 300 python tools/pdl_ab.py --configs c4_2048x512_s80,c4_512x2048_s80,c4_2048x512_s95,c4_512x2048_s95,c3_512x512 >> gpurun_out/ro_ab.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_pdl.py tests/test_gpu_serialize.py tests/test_gpu_guards.py -m gpu -q -x > gpurun_out/ro_pytest.log 2>&1
tail -1 gpurun_out/ro_build.log; cat gpurun_out/ro_ab.log; tail -3 gpurun_out/ro_pytest.log
