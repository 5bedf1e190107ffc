# ncu --set full of the bench's other legs' top kernels: k_dense_tc (A8) and the screen-space
# rasters (f1); summaries via tools/screen_summary.py / profiles/r02_dense_tc.md
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_dense_tc|k_dense_bwd" -c 2 \
  -o gpurun_out/r02_dense_full python tools/dense_case.py > gpurun_out/r02_dense_full.log 2>&1; echo dense rc=$?
STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sraster" -c 3 \
  -o gpurun_out/r02_screen_full python tools/screen_case.py > gpurun_out/r02_screen_full.log 2>&1; echo screen rc=$?
