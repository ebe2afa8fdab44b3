python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pt_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pdl.py tests/test_gpu_conv.py -m gpu -q > gpurun_out/pt_pytest.log 2>&1
tail -5 gpurun_out/pt_pytest.log
