python tools/prof_conv.py 256 7 8 0.9 > gpurun_out/prof_conv_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv2 -c 1 -o gpurun_out/conv2_256_7 python tools/prof_conv.py 256 7 8 0.9 > gpurun_out/ncu_conv.log 2>&1
