python tools/prof_conv.py 256 28 8 0.9 > gpurun_out/prof_conv3_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv2 -c 1 -o gpurun_out/conv2_256_28 python tools/prof_conv.py 256 28 8 0.9 > gpurun_out/ncu_conv3.log 2>&1
