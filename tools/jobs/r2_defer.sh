# TMEM-R issuer: deferred slot refill (DEFER=1, product default) vs waiting for the copies just issued (DEFER=0),
# ring depth 8 / 16 pieces; graph-timed configs (tools/pdl_ab.py) + c5 bench lines, same box, two rounds
rm -f gpurun_out/defer_*
run() {  # $1 label
  timeout 300 python tools/pdl_ab.py | sed "s/^/$1 /" >> gpurun_out/defer_ab.log 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --no-proxy --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^/$1 /" >> gpurun_out/defer_ab.log
}
for i in 1 2; do
  python paper_2101_07948_b200/build.py --force >> gpurun_out/defer_build.log 2>&1; run D1P8
  SDNN_NVCC_FLAGS="-DSDNN_TMEMR_DEFER=0" python paper_2101_07948_b200/build.py --force >> gpurun_out/defer_build.log 2>&1; run D0P8
  SDNN_NVCC_FLAGS="-DSDNN_TMEMR_PIECES=16" python paper_2101_07948_b200/build.py --force >> gpurun_out/defer_build.log 2>&1; run D1P16
done
python paper_2101_07948_b200/build.py --force >> gpurun_out/defer_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jitter.py tests/test_gpu_pdl.py -m gpu -q -x > gpurun_out/defer_pytest.log 2>&1
tail -3 gpurun_out/defer_pytest.log
python - <<'PY'
import json, collections
rows = collections.defaultdict(list)
for line in open("gpurun_out/defer_ab.log"):
    lab, _, js = line.partition(" ")
    try: d = json.loads(js)
    except Exception: continue
    key = d.get("config") if "us" in d or "us_per_pair" in d else "c5_bench_ms"
    if isinstance(key, dict): key = "c5_bench_ms"
    v = d.get("us", d.get("us_per_pair", d.get("ms_per_step")))
    rows[(key, lab)].append(v)
keys = sorted({k for k, _ in rows})
for k in keys:
    print(f"{k:32s}", "  ".join(f"{lab} {min(rows[(k, lab)]):9.2f}" for lab in ("D0P8", "D1P8", "D1P16") if (k, lab) in rows))
PY
