CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_v6.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smooth_up -s 8 -c 1 -o gpurun_out/prof_v6_up $CMD > gpurun_out/ncu_v6a.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:pcg_apply -s 3 -c 1 -o gpurun_out/prof_v6_ap $CMD > gpurun_out/ncu_v6b.log 2>&1
tail -1 gpurun_out/ncu_v6a.log gpurun_out/ncu_v6b.log
