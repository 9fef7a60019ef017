set -x
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_v1.json 2> gpurun_out/plain_v1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_v1.csv $CMD > gpurun_out/ncu_launch_v1.log 2>&1
$CMD > gpurun_out/plain_v1b.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pcg_apply -s 20 -c 2 -o gpurun_out/prof_v1 $CMD > gpurun_out/ncu_full_v1.log 2>&1
ls -la gpurun_out
