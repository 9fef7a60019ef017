# bench (profiling restricted to the dominant kernel in the timed region) + GPU suite
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_b.json')); k=d['kernels_ms_profiled_step']
print('value', round(d['value'],1), 'ms/step', d['ms_per_step'], 'sum kernels (profiled step)', round(sum(k.values()),1), d['clocks'])
print(d['roofline'])"
tail -3 gpurun_out/bench_b.err
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_b.log
