# CTA-local split-row pieces (summed in shared memory by the row kernel) vs workspace + split_reduce_kernel
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/loc_build.log 2>&1
for i in 1 2; do
SDNN_LOCAL_PIECES=0 timeout 300 python tools/pdl_ab.py --configs c1,c2_768x768,c2_3072x768,c2_768x3072,c3_128x64 >> gpurun_out/loc_ab.log 2>&1
timeout 300 python tools/pdl_ab.py --configs c1,c2_768x768,c2_3072x768,c2_768x3072,c3_128x64 >> gpurun_out/loc_ab.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/loc_pytest.log 2>&1
cat gpurun_out/loc_ab.log; tail -3 gpurun_out/loc_pytest.log; tail -1 gpurun_out/loc_build.log
