#!/bin/bash
# one gpurun call: GPU parity tests + a short bench; logs under gpurun_out/
TAG=${1:-x}
timeout 1000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_$TAG.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests_$TAG.log
timeout 300 python bench.py --steps 20 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$TAG.log 2>&1; echo exit=$? >> gpurun_out/bench_$TAG.log
if [ -n "$BENCH_SEP" ]; then
  timeout 300 python bench.py --steps 20 --warmup 3 --separate --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_sep_$TAG.log 2>&1; echo exit=$? >> gpurun_out/bench_sep_$TAG.log
fi
