timeout 300 python tools/bench_configs.py --configs c1,c2_768x768,c2_768x3072,c3_128x64,c3_256x128,c2_3072x768,c3_512x512 --variants row,auto --graph --iters 10 2>/dev/null
timeout 200 python tools/time_cfg.py --config c5 --kernel row
timeout 600 python -m pytest tests -m gpu -q -x -k "row or auto or ragged or degenerate or unaligned or graph or host" 2>&1 | tail -2
