# round 2: new GPU tests (shards, corrupt blobs, tune), bench default line, ncu full capture of the bench kernel
timeout 900 python -m pytest tests/test_gpu_shards.py tests/test_gpu_serialize.py -q -s 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "tune" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; tail -c 6000 gpurun_out/r2_bench.log
python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tmemr -s 1 -c 1 -o gpurun_out/r2_tmemr_full python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/r2_ncu.log 2>&1
tail -3 gpurun_out/r2_ncu.log
