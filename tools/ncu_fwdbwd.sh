# one --set full capture of k_fwdbwd and k_query (source-level), plus the launch list of a short bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fwdbwd|k_query" --launch-skip 6 --launch-count 2 \
  -f -o gpurun_out/r02_eval_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-screen --no-general --no-graph --clock-window 0 \
  > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-screen --no-general --clock-window 0 \
  > gpurun_out/ncu_list.log 2>&1; echo list rc=$?
