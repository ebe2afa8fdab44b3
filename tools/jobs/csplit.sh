for m in 16 4; do SDNN_CONV_SPLIT_MIN=$m timeout 600 python tools/conv_bench.py --sizes 32,64,128 --images 7,14,28 > gpurun_out/csplit_$m.log 2>&1; done
