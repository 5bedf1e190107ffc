# one gpurun call: build, round-2 + round-1 GPU parity tests, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity_r2.py -q -m gpu > gpurun_out/r2tests.log 2>&1; echo r2 rc=$?
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/r1tests.log 2>&1; echo r1 rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -n 3 gpurun_out/r2tests.log gpurun_out/r1tests.log
