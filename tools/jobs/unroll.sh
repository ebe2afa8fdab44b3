VARIANTS="A U2 U4" bash tools/jobs/abn.sh
VARIANTS="A U2 U4" KERN=tmem8 bash tools/jobs/abn.sh
VARIANTS="A U2 U4" CFG=c4_2048x512_s80 KERN=auto ITERS=20 bash tools/jobs/abn.sh
