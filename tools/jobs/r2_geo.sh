python -c "import __graft_entry__ as g; g.build()" > gpurun_out/geo_build.log 2>&1
for st in "" 2 3 4; do SDNN_ROW_STAGES=$st timeout 300 python tools/c2_geo.py >> gpurun_out/geo.log 2>&1; done
cat gpurun_out/geo.log
