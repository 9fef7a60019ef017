timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "solve_vs_oracle or galerkin_fewer or cfg4 or level_draws" > gpurun_out/pytest_surr.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_surr.log
for v in base surr3; do
  case $v in base) ENV="";; *) ENV="OSC_LIB=$PWD/ab/$v.so";; esac
  env $ENV timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_surr_$v.json 2> gpurun_out/bench_surr_$v.err; echo "$v exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_surr_$v.json')); k=d['kernels_ms_profiled_step']; g=d['kernel_gbs']
print('$v value', round(d['value'],1), 'sum', round(sum(k.values()),1), d['clocks']['sm_mhz'], {n: (k[n], g.get(n)) for n in k if 'smooth_up' in n})"
done
