# SURVEY §8(d) counters: one ncu-profiled call per config (auto kernel), every kernel of the call
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_inst_executed_op_tmem_ldt.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,launch__grid_size,launch__registers_per_thread
mkdir -p gpurun_out/cfgncu
for c in c1 c2_768x768 c2_3072x768 c2_768x3072 c3_128x64 c3_256x128 c3_512x512 c3_1024x512 c4_2048x512_s80 c4_512x2048_s80 c4_2048x512_s95 c4_512x2048_s95; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:'spmm|split' --csv --log-file gpurun_out/cfgncu/$c.csv \
    python tools/prof_one.py --config $c --kernel auto --launches 1 > gpurun_out/cfgncu/$c.log 2>&1
done
timeout 300 ncu --metrics $M --clock-control none -k regex:'spmm|split' --csv --log-file gpurun_out/cfgncu/c5_n65536.csv \
  python tools/prof_one.py --config c5 --kernel auto --n 65536 --launches 1 > gpurun_out/cfgncu/c5.log 2>&1
