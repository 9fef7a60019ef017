timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "solver_variants" > gpurun_out/pytest_var.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_var.log
for v in base xi8; do
  case $v in base) ENV="";; *) ENV="OSC_LIB=$PWD/ab/$v.so";; esac
  env $ENV timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xi_$v.json 2> gpurun_out/bench_xi_$v.err; echo "$v exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_xi_$v.json')); print('$v', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
