# round 2: full GPU suite + smoke + c5 timing
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python tools/time_cfg.py --config c5 --kernel tmem --n 65536 --iters 5 2>&1
