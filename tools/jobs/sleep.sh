VARIANTS="A S1 S2" bash tools/jobs/abn.sh
VARIANTS="A S1 S2" CFG=c4_2048x512_s80 KERN=auto ITERS=20 bash tools/jobs/abn.sh
