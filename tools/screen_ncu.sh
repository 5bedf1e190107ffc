# launch list of the screen-space leg alone (gc_render + gc_fit_image at 1920x1080, cfg2)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/screen_case.py > gpurun_out/screen_case.txt 2>&1
STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/screen_launches.csv python tools/screen_case.py > gpurun_out/screen_ncu.log 2>&1; echo rc=$?
