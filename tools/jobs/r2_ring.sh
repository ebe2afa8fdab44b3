# TMEM-R smem ring depth: 16 pieces (4 K chunks of X in flight) vs 8 (2 chunks), same box
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ring_build.log 2>&1
for i in 1 2; do
timeout 300 python tools/pdl_ab.py | sed 's/^/R16 /' >> gpurun_out/ring_ab.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-proxy --e2e-steps 1 2>/dev/null | tail -1 | sed 's/^/R16 /' >> gpurun_out/ring_ab.log
done
SDNN_NVCC_FLAGS="-DSDNN_TMEMR_PIECES=8" python paper_2101_07948_b200/build.py --force >> gpurun_out/ring_build.log 2>&1
for i in 1 2; do
timeout 300 python tools/pdl_ab.py | sed 's/^/R8 /' >> gpurun_out/ring_ab.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-proxy --e2e-steps 1 2>/dev/null | tail -1 | sed 's/^/R8 /' >> gpurun_out/ring_ab.log
done
python paper_2101_07948_b200/build.py --force >> gpurun_out/ring_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_pdl.py tests/test_gpu_serialize.py -m gpu -q -x > gpurun_out/ring_pytest.log 2>&1
tail -3 gpurun_out/ring_pytest.log
