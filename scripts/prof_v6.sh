CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_v11.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smooth_up -s 8 -c 1 -o gpurun_out/prof_v11_up $CMD > gpurun_out/ncu_v11a.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:update_down -s 3 -c 1 -o gpurun_out/prof_v11_ud $CMD > gpurun_out/ncu_v11b.log 2>&1
tail -1 gpurun_out/ncu_v11a.log gpurun_out/ncu_v11b.log
