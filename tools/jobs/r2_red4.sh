# float4 split-K reduction: configs graph-timed + parity / jitter / pdl / conv tests
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r5_build.log 2>&1
timeout 300 python tools/pdl_ab.py > gpurun_out/r5_ab.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_pdl.py tests/test_gpu_conv.py tests/test_gpu_gather.py -m gpu -q -x > gpurun_out/r5_pytest.log 2>&1
tail -1 gpurun_out/r5_build.log; cat gpurun_out/r5_ab.log; tail -3 gpurun_out/r5_pytest.log
