# level-0 ring kernels: GPU suite, bench ring vs register-prefetch, ncu of the two ring kernels
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_l0r.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_l0r.log
for v in ring noring; do
  case $v in ring) ENV="";; noring) ENV="OSC_L0_RING=0";; esac
  env $ENV timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_l0r_$v.json 2> gpurun_out/bench_l0r_$v.err; echo "$v exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_l0r_$v.json')); k=d['kernels_ms_profiled_step']; g=d['kernel_gbs']
print('$v value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'sum', round(sum(k.values()),1), 'iters', d['config']['mean_iters_fine'], d['clocks']['sm_mhz'])
print({n: (k[n], g.get(n)) for n in k if '@2048' in n and ('pcg' in n or '.L0' in n)})"
done
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
for spec in "smooth_up_ring_kernel 2" "restrict_ring_kernel 2"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_l0_$1 $CMD > gpurun_out/ncu_l0_$1.log 2>&1
  tail -1 gpurun_out/ncu_l0_$1.log
done
