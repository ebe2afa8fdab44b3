# c2 768² probe: plan / geometry knobs, env knobs, ncu launch list of the auto call
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2p_build.log 2>&1
for e in "" "SDNN_ROW_V=2" "SDNN_ROW_V=4" "SDNN_SPLIT_K=2" "SDNN_SPLIT_K=4" "SDNN_ROW_STAGES=1" "SDNN_ROW_STAGES=2" "SDNN_ROW_STAGES=3"; do
  env $e timeout 200 python tools/c2_probe2.py >> gpurun_out/c2p.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"spmm|reduce" -c 6 --csv python tools/c2_probe2.py --variants auto > gpurun_out/c2p_ncu.csv 2>&1
cat gpurun_out/c2p.log
