CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_f.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_f.csv $CMD > gpurun_out/ncu_launch_f.log 2>&1
for spec in "update_down 2" "pcg_apply 2" "smooth_up_kernel 5" "restrict_kernel 0" "sub_vcycle 0"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_f_$1 $CMD > gpurun_out/ncu_f_$1.log 2>&1
  tail -1 gpurun_out/ncu_f_$1.log
done
