# round-2 check (session 2, after the second TMEM plan): smoke, GPU suite, bench, reference arm, launch list, full capture
# ncu launch list of the bench command, ncu --set full of the bench kernel (c5, N = 65536)
rm -f gpurun_out/f4_*
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f4_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f4_pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/f4_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f4_bench_ref.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-proxy > gpurun_out/f4_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f4_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-proxy > gpurun_out/f4_ncu_bench.log 2>&1
python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/f4_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tmemr -s 1 -c 1 -o gpurun_out/f4_tmemr_full python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/f4_ncu_full.log 2>&1
tail -2 gpurun_out/f4_smoke.log; tail -2 gpurun_out/f4_pytest.log; tail -c 400 gpurun_out/f4_bench.log; tail -c 300 gpurun_out/f4_bench_ref.log; tail -2 gpurun_out/f4_ncu_full.log
