timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py -m gpu -q -x -k "chain or permuted or narrow or multi or smoke or config_parity" 2>&1 | tail -3
timeout 600 python tools/chain_bench.py > gpurun_out/chain_bench.jsonl 2> gpurun_out/chain_bench.err
