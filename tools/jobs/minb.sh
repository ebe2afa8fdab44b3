for v in A M2 M3; do SDNN_PKG_DIR=ab/$v timeout 600 python tools/conv_bench.py --sizes 64,128,256 --images 14,28,56 > gpurun_out/minb_$v.log 2>&1; done
