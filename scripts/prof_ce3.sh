CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_ce3.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ce_rows -s 2 -c 1 -o gpurun_out/prof_ce3r $CMD > gpurun_out/ncu_ce3.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:ce_cols -s 2 -c 1 -o gpurun_out/prof_ce3c $CMD >> gpurun_out/ncu_ce3.log 2>&1
tail -1 gpurun_out/ncu_ce3.log
