set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r1_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench_auto.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --kernel codegen --no-cpu-baseline > gpurun_out/r1_bench_cg.log 2>&1
timeout 600 python tools/bench_configs.py --variants row,codegen > gpurun_out/r1_configs.jsonl 2>gpurun_out/r1_configs.err
