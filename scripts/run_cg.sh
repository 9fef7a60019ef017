# one-reduction PCG: GPU suite, bench new vs legacy, launch-bound variants
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_cg.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_cg.log
for v in new legacy sur4 rr4; do
  case $v in
    new) ENV="";; legacy) ENV="OSC_LEGACY_PCG=1";; *) ENV="OSC_LIB=$PWD/ab/$v.so";;
  esac
  env $ENV timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cg_$v.json 2> gpurun_out/bench_cg_$v.err; echo "$v exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_cg_$v.json')); k=d['kernels_ms_profiled_step']; g=d['kernel_gbs']
print('$v value', round(d['value'],1), 'iters', d['config']['mean_iters_fine'], d['config']['mean_iters_coarse'], d['clocks']['sm_mhz'])
print({n: (k[n], g.get(n)) for n in k if '@2048' in n and ('pcg' in n or '.L0' in n)})"
  tail -2 gpurun_out/bench_cg_$v.err
done
