python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rp_build.log 2>&1
timeout 900 python tools/tmem_rows_probe.py > gpurun_out/rp.log 2>&1
cat gpurun_out/rp.log
