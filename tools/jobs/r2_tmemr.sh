# round 2: replicated-quarter TMEM kernel — parity subset, c5 timing, bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/time_cfg.py --config c5 --kernel tmem,tmem8,row --n 65536 --iters 5 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "tmem or auto or smoke" 2>&1 | tail -15
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
