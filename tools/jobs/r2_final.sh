# round-2 check: build, smoke, full GPU suite, bench (default + reference arm), allgather flag at N=1
rm -f gpurun_out/fc2_*
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fc2_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fc2_pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/fc2_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fc2_bench_ref.log 2>&1
timeout 300 python bench.py --gpus 1 --steps 5 --warmup 3 --allgather --no-cpu-baseline --no-configs --no-proxy > gpurun_out/fc2_bench_ag.log 2>&1
tail -3 gpurun_out/fc2_pytest.log; tail -2 gpurun_out/fc2_smoke.log
