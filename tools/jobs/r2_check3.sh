# round-2 re-entry check: build, smoke, full GPU suite, bench
rm -f gpurun_out/c3_*
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c3_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/c3_pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/c3_bench.log 2>&1
tail -3 gpurun_out/c3_pytest.log; tail -2 gpurun_out/c3_smoke.log; tail -c 600 gpurun_out/c3_bench.log
