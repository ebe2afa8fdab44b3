for wc in 0 2 1; do timeout 600 python tools/conv_bench.py --cta-panels $wc --sizes 64,256 --images 7,14,28 > gpurun_out/conv_wc$wc.log 2>&1; done
