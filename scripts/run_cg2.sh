# lagged convergence polling: GPU suite + repeated benches (timed-region gap vs profiled kernel sum)
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_cg2.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_cg2.log
for i in 1 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cg2_$i.json 2> gpurun_out/bench_cg2_$i.err; echo "run $i exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_cg2_$i.json')); k=d['kernels_ms_profiled_step']
print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'kernel sum', round(sum(k.values()),1), d['clocks'], 'launches', d['gpu_launches'])"
done
