python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p5_build.log 2>&1
for i in 1 2; do
for P in 0 1; do SDNN_TMEM_PERSIST=$P timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-proxy --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^/P$P /" >> gpurun_out/p5.log; done
done
cut -c1-200 gpurun_out/p5.log
