VARIANTS="A R RD" bash tools/jobs/abn.sh
VARIANTS="A R RD" CFG=c3_512x512 KERN=auto ITERS=50 bash tools/jobs/abn.sh
