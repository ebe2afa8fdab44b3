# refresh: sparse conv suite vs cuDNN dense, chained FFN pair
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cc_build.log 2>&1
timeout 900 python tools/conv_bench.py --out gpurun_out/r2s2_conv_bench.jsonl > gpurun_out/r2s2_conv.log 2>&1
timeout 600 python tools/chain_bench.py > gpurun_out/r2s2_chain.jsonl 2>&1
tail -3 gpurun_out/r2s2_conv.log; tail -3 gpurun_out/r2s2_chain.jsonl
