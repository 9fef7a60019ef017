# coarse V-cycle kernels: level stats bench (mode 2), GPU suite, ncu of the ring kernels at level 1 of 2048^2
OSC_LEVEL_STATS=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cmx.json 2> gpurun_out/bench_cmx.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cmx.json')); k=d['kernels_ms']; g=d['kernel_gbs']
print('value', round(d['value'],1), 'iters', d['config']['mean_iters_fine'], d['config']['mean_iters_coarse'])
print({n: (k[n], g.get(n)) for n in k if '@2048' in n and ('mg_up' in n or 'mg_down' in n)})"
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_cm.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_cm.log
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
for spec in "c_up_ring 4" "c_down_ring 0"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_r2_$1 $CMD > gpurun_out/ncu_r2_$1.log 2>&1
  tail -1 gpurun_out/ncu_r2_$1.log
done
