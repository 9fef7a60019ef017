# nested iteration (coarse coupled solve prolonged as the fine PCG's start): GPU suite; bench vs OSC_NO_NESTED
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_nested.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_nested.log
for v in nested plain; do
  case $v in plain) ENV="OSC_NO_NESTED=1";; *) ENV="";; esac
  env $ENV timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_nest_$v.json 2> gpurun_out/bench_nest_$v.err; echo "$v exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_nest_$v.json'))
print('$v value', round(d['value'],1), 'iters', d['config']['mean_iters_fine'], d['config']['mean_iters_coarse'], d['clocks']['sm_mhz'])"
  env $ENV timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_nest_c3_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_nest_c3_$v.json'))
print('$v cfg3', round(d['value'],1), 'iters', d['config']['mean_iters_fine'], d['config']['mean_iters_coarse'])"
done
