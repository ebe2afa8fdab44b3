timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python tools/bench_configs.py --variants auto --graph > gpurun_out/tsk_cfg.jsonl 2> gpurun_out/tsk_cfg.err
timeout 1200 python tools/sweep.py --out gpurun_out/sweep6.jsonl > gpurun_out/sweep6.log 2>&1
