set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/refresh_round.sh final
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-general --clock-window 0 \
  > gpurun_out/final_ncu_list.log 2>&1; echo list rc=$?
tail -n 2 gpurun_out/final_default.log gpurun_out/final_cfg4.log gpurun_out/final_reference.log
