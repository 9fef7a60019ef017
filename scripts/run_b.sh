# fused setup: targeted tests, bench, full GPU suite
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fused_setup or galerkin_fewer or solve_vs_oracle" > gpurun_out/pytest_fs.log 2>&1; echo "pytest-fs exit $?"; tail -15 gpurun_out/pytest_fs.log
OSC_LEVEL_STATS=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fs.json 2> gpurun_out/bench_fs.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_fs.json')); k=d['kernels_ms_profiled_step']
print('value', round(d['value'],1), 'ms/step', d['ms_per_step'], 'iters', d['config']['mean_iters_fine'], d['config']['mean_iters_coarse'], d['clocks'])
print({n: v for n, v in k.items() if 'setup' in n})"
tail -3 gpurun_out/bench_fs.err
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_b.log
