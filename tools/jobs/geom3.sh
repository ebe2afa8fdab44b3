for c in c2_768x3072 c2_768x768 c3_512x512 c3_256x128 c2_3072x768; do
  for o in "" panel_rows=8,cta_panels=4 panel_rows=4,cta_panels=8 panel_rows=8,cta_panels=8 panel_rows=4,cta_panels=16 panel_rows=8,cta_panels=16; do
    timeout 120 python tools/time_cfg.py --config $c --kernel row --opts "$o" --iters 30
  done
done
