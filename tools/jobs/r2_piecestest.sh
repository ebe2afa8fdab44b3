python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pc_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pieces.py -m gpu -q > gpurun_out/pc_pytest.log 2>&1
tail -5 gpurun_out/pc_pytest.log
