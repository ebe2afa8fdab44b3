#!/bin/bash
# c4 at 95 %: TMEM (auto) vs row-plan geometries (taller CTAs share one staged X tile).
mkdir -p gpurun_out; rm -f gpurun_out/c4_95.log
for cfg in c4_2048x512_s95 c4_512x2048_s95; do
  python tools/time_cfg.py --config $cfg --kernel auto,tmem,tmem8,row --iters 20 >> gpurun_out/c4_95.log 2>&1
  for o in panel_rows=8,cta_panels=16 panel_rows=8,cta_panels=24 panel_rows=8,cta_panels=31 panel_rows=4,cta_panels=31 panel_rows=8,cta_panels=8; do
    python tools/time_cfg.py --config $cfg --kernel row --opts $o --iters 20 >> gpurun_out/c4_95.log 2>&1
  done
  python tools/time_cfg.py --config $cfg --kernel group --iters 20 >> gpurun_out/c4_95.log 2>&1
done
