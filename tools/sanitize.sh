# compute-sanitizer memcheck / racecheck / synccheck of tools/sanitize_case.py; summaries in gpurun_out/
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -n 4 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
