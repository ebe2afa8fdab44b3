# full GPU check: build, smoke, GPU tests, bench, ncu launch list of the bench command, full capture
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/rc_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rc_pytest.log 2>&1
timeout 400 python bench.py > gpurun_out/rc_bench.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/rc_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rc_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/rc_ncu.log 2>&1
python tools/prof_one.py --config c5 --kernel auto --n 65536 > gpurun_out/rc_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tmem -s 1 -c 1 -o gpurun_out/rc_tmem_full python tools/prof_one.py --config c5 --kernel auto --n 65536 > gpurun_out/rc_ncu2.log 2>&1
timeout 600 python tools/bench_configs.py --variants auto,row,tmem --graph > gpurun_out/rc_cfg.jsonl 2> gpurun_out/rc_cfg.err
