# PDL A/B: graph-timed c1-c4 + dependent FFN chain with and without programmatic dependent launch
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pdl_build.log 2>&1
SDNN_PDL=0 timeout 300 python tools/pdl_ab.py > gpurun_out/pdl_ab.log 2>&1
timeout 300 python tools/pdl_ab.py >> gpurun_out/pdl_ab.log 2>&1
SDNN_PDL=0 timeout 300 python tools/pdl_ab.py >> gpurun_out/pdl_ab.log 2>&1
timeout 300 python tools/pdl_ab.py >> gpurun_out/pdl_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_chain.py -m gpu -q -x > gpurun_out/pdl_pytest.log 2>&1
cat gpurun_out/pdl_ab.log; tail -3 gpurun_out/pdl_pytest.log
