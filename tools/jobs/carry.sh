timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
VARIANTS="A B" bash tools/jobs/abn.sh
VARIANTS="A B" KERN=tmem8 bash tools/jobs/abn.sh
for c in c4_2048x512_s80 c4_512x2048_s95 c3_512x512 c2_3072x768; do VARIANTS="A B" CFG=$c KERN=auto ITERS=20 bash tools/jobs/abn.sh; done
