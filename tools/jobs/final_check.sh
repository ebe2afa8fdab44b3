# round-end check: build, smoke, full GPU suite, bench (default + reference arm + allgather flag at N=1),
# ncu launch list of the bench command, per-config timings
rm -f gpurun_out/fc_*
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fc_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fc_pytest.log 2>&1
timeout 400 python bench.py > gpurun_out/fc_bench.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fc_bench_ref.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fc_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fc_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fc_ncu.log 2>&1
timeout 900 python tools/bench_configs.py --variants auto --graph > gpurun_out/fc_cfg.jsonl 2> gpurun_out/fc_cfg.err
