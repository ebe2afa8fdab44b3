# row-plan geometry vs small N (one N tile): rows per CTA = panel_rows × cta_panels
for shape in 4096x4096:0.9 2048x2048:0.9 1024x1024:0.9 4096x4096:0.7; do
  for o in "" panel_rows=8,cta_panels=8 panel_rows=4,cta_panels=8 panel_rows=4,cta_panels=4 panel_rows=8,cta_panels=4 panel_rows=4,cta_panels=2; do
    for n in 128 256 512; do
      timeout 120 python tools/time_cfg.py --shape $shape --n $n --kernel row --opts "$o" --iters 20
    done
  done
done
