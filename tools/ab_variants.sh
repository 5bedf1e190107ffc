# A/B of library variants on one box: VARIANTS="base noatom ..." (gpurun_var_<name>.so; base = in-tree)
cp paper_2507_19718_b200/libgscache.so gpurun_var_base.so
for rep in 1 2; do
for v in $VARIANTS; do
  cp gpurun_var_$v.so paper_2507_19718_b200/libgscache.so
  timeout 600 python bench.py ${BENCH_ARGS:---steps 30 --warmup 5} --no-cpu-baseline --no-general --no-screen --no-dense --clock-window 0 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "
import json,sys;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]);pk=d['roofline']['per_kernel']
print('$v', round(d['ms_per_step']*1e3,1), ' '.join(f'{k}={v[\"ms\"]*1e3:.1f}' for k,v in pk.items()))"
done; done
cp gpurun_var_base.so paper_2507_19718_b200/libgscache.so
