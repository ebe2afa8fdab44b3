# full GPU suite + smoke + bench (default line)
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2_bench2.log 2>&1; tail -c 3000 gpurun_out/r2_bench2.log
