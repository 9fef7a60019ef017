timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_v16.json 2> gpurun_out/bench_v16.err; echo "bench exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_v16.json')); print(d['value'], d['config']['mean_iters_fine']); print(d['kernels_ms'])"; tail -2 gpurun_out/bench_v16.err
CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_ce.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ce_rows|ce_cols" -s 2 -c 2 -o gpurun_out/prof_ce2 $CMD > gpurun_out/ncu_ce.log 2>&1
tail -1 gpurun_out/ncu_ce.log
