CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_r1.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch_r1.log 2>&1
$CMD > gpurun_out/plain_r1b.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"update_down|smooth_up|pcg_apply|restrict_kernel" -s 40 -c 8 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full_r1.log 2>&1
tail -1 gpurun_out/ncu_launch_r1.log gpurun_out/ncu_full_r1.log
