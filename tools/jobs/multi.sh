timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "multi or split or config_parity or graph or host" 2>&1 | tail -3
bash tools/jobs/ab.sh
CFG=c2_768x768 KERN=row ITERS=50 bash tools/jobs/ab.sh
CFG=c4_2048x512_s80 KERN=auto ITERS=20 bash tools/jobs/ab.sh
