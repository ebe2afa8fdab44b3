# TMEM-R bridge format (odd row segments paired with the next row's first entry): bench c5, configs, full GPU suite
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/br_build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/br_bench.log 2>&1
timeout 300 python tools/pdl_ab.py > gpurun_out/br_ab.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/br_pytest.log 2>&1
tail -1 gpurun_out/br_build.log; tail -c 1500 gpurun_out/br_bench.log; cat gpurun_out/br_ab.log; tail -3 gpurun_out/br_pytest.log
