for ks in 0 2 4 6; do SDNN_SPLIT_K=$ks timeout 200 python tools/c2_probe.py; done
