# screen-space leg: parity tests, timing, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_screen.py -x -q > gpurun_out/screen_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/screen_tests.log
for i in 1 2 3; do timeout 300 python tools/screen_case.py 2>&1 | tail -1; done
STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/screen_launches.csv python tools/screen_case.py > gpurun_out/screen_ncu.log 2>&1; echo ncu rc=$?
