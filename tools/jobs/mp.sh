timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config_parity and tmem" 2>&1 | tail -2
VARIANTS="B MP" bash tools/jobs/abn.sh
VARIANTS="B MP" KERN=tmem8 bash tools/jobs/abn.sh
VARIANTS="B MP" CFG=c4_2048x512_s80 KERN=auto ITERS=20 bash tools/jobs/abn.sh
VARIANTS="B MP" CFG=c3_1024x512 KERN=auto ITERS=20 bash tools/jobs/abn.sh
