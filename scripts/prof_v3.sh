CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_v3.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"smooth_up|pcg_update_down|pcg_apply|restrict_kernel" -s 40 -c 4 -o gpurun_out/prof_v3 $CMD > gpurun_out/ncu_full_v3.log 2>&1
tail -3 gpurun_out/ncu_full_v3.log
