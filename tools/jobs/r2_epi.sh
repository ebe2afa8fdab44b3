# TMEM-R epilogue: output rows / biases loaded once per warp (lane-distributed) instead of per row
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/epi2_build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-proxy > gpurun_out/epi2_bench.log 2>&1
timeout 300 python tools/pdl_ab.py > gpurun_out/epi2_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_gather.py tests/test_gpu_chain.py tests/test_gpu_serialize.py tests/test_gpu_shards.py -m gpu -q -x > gpurun_out/epi2_pytest.log 2>&1
tail -1 gpurun_out/epi2_build.log; python -c "
import json;l=[x for x in open('gpurun_out/epi2_bench.log') if x.startswith('{')];d=json.loads(l[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['design_ceiling']['frac_of_design_ceiling'])"; cat gpurun_out/epi2_ab.log; tail -3 gpurun_out/epi2_pytest.log
