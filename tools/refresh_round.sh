#!/bin/bash
# end-of-milestone evidence refresh (one gpurun call; no ncu here):
#   default bench line, reference arm, cfg4 line, parity report, frame timeline
TAG=${1:-final}
timeout 600 python bench.py > gpurun_out/${TAG}_default.log 2>&1; echo exit=$? >> gpurun_out/${TAG}_default.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_reference.log 2>&1; echo exit=$? >> gpurun_out/${TAG}_reference.log
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4.log 2>&1; echo exit=$? >> gpurun_out/${TAG}_cfg4.log
timeout 900 python tests/parity_report.py > gpurun_out/${TAG}_parity.json 2> gpurun_out/${TAG}_parity.err; echo exit=$? >> gpurun_out/${TAG}_parity.err
timeout 300 python tools/timeline.py --graph --frames 3 > gpurun_out/${TAG}_timeline.txt 2>&1
