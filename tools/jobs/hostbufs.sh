timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k host 2>&1 | tail -1
for r in 1 2; do for v in H2 H3 H4; do SDNN_PKG_DIR=ab/$v timeout 300 python tools/e2e_blocks.py --blocks 0,8192 2>&1 | grep block_cols | sed "s/^/$v /"; done; done
