CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_v4.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smooth_up -s 30 -c 1 -o gpurun_out/prof_v4_up $CMD > gpurun_out/ncu_v4a.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:update_down -s 30 -c 1 -o gpurun_out/prof_v4_ud $CMD > gpurun_out/ncu_v4b.log 2>&1
tail -2 gpurun_out/ncu_v4a.log gpurun_out/ncu_v4b.log
