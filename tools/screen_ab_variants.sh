# screen-space leg A/B of library variants on one box: VARIANTS="base prev" (gpurun_var_<name>.so; base = in-tree)
cp paper_2507_19718_b200/libgscache.so gpurun_var_base.so
for rep in 1 2; do
for v in $VARIANTS; do
  cp gpurun_var_$v.so paper_2507_19718_b200/libgscache.so
  echo "$v $(timeout 300 python tools/screen_case.py 2>&1 | tail -1)"
done; done
cp gpurun_var_base.so paper_2507_19718_b200/libgscache.so
