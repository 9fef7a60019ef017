# per-level kernel times (no profiler) + ncu --set full of the coarse-level 9-point kernels at level 1 of 2048^2
OSC_LEVEL_STATS=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_lvl.json 2> gpurun_out/bench_lvl.err; echo "lvl exit $?"
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_c.json 2>&1 || exit 1
for spec in "c_up_march 4" "c_restrict_march 0" "c_pre_march 0" "rap_kernel 0" "prow_kernel 0"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_c_$1 $CMD > gpurun_out/ncu_c_$1.log 2>&1
  tail -1 gpurun_out/ncu_c_$1.log
done
