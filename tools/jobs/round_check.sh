# full GPU check: build, smoke, GPU tests, bench, ncu launch list of the bench command
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/rc_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rc_pytest.log 2>&1
timeout 400 python bench.py > gpurun_out/rc_bench.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/rc_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rc_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/rc_ncu.log 2>&1
