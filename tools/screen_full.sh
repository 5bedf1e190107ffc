# ncu --set full of the screen-space raster kernels (forward with fused loss, backward)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
STEPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sraster_bwd" -c 1 \
  -o gpurun_out/screen_bwd python tools/screen_case.py > gpurun_out/screen_full.log 2>&1; echo rc=$?
