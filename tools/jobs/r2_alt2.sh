# auto handles with a second TMEM plan (~25 % more row blocks) picked per call: configs, c5, tests
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/a2_build.log 2>&1
timeout 300 python tools/pdl_ab.py > gpurun_out/a2_ab.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-proxy --e2e-steps 1 2>/dev/null | tail -1 >> gpurun_out/a2_ab.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_pdl.py tests/test_gpu_serialize.py tests/test_gpu_conv.py tests/test_gpu_chain.py tests/test_gpu_gather.py -m gpu -q -x > gpurun_out/a2_pytest.log 2>&1
tail -1 gpurun_out/a2_build.log; cut -c1-300 gpurun_out/a2_ab.log; tail -3 gpurun_out/a2_pytest.log
