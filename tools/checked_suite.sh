# Bounds-checked build (-DGSC_CHECKED: device-side checks that trap on any out-of-range index in
# the hot kernels; compute-sanitizer is refused on this GPU pool) under the whole -m gpu suite,
# smoke() and the randomised API soak.  One gpurun call:
#   python tools/build_variant.py gpurun_var_checked.so -DGSC_CHECKED=1   (here, first)
#   gpurun -- 'bash tools/checked_suite.sh'
set -x
cp paper_2507_19718_b200/libgscache.so /tmp/libgscache.product.so
cp gpurun_var_checked.so paper_2507_19718_b200/libgscache.so
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/checked_tests.log 2>&1; echo tests rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/checked_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python tests/fuzz_api.py --calls 1500 --seed 5 > gpurun_out/checked_fuzz.log 2>&1; echo fuzz rc=$?
cp /tmp/libgscache.product.so paper_2507_19718_b200/libgscache.so
tail -n 3 gpurun_out/checked_tests.log gpurun_out/checked_smoke.log gpurun_out/checked_fuzz.log
grep -h "GSC_CHECK failed" gpurun_out/checked_*.log | sort | uniq -c | head
