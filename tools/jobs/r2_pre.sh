# after the producer offset batching + epilogue prefetch: graph-timed configs, parity subset
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/pre_build.log 2>&1
timeout 300 python tools/pdl_ab.py > gpurun_out/pre_ab.log 2>&1
timeout 300 python tools/pdl_ab.py >> gpurun_out/pre_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_chain.py tests/test_gpu_guards.py -m gpu -q -x > gpurun_out/pre_pytest.log 2>&1
cat gpurun_out/pre_ab.log; tail -3 gpurun_out/pre_pytest.log; tail -1 gpurun_out/pre_build.log
