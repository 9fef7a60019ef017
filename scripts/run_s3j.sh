# geometric host-xi chunks: parity tests + e2e A/B on cfg4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "host_xi or slot or level_draws or cfg4" > gpurun_out/pytest_s3j.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3j.log
for rep in 1 2; do
for v in geom equal; do
  case $v in equal) ENV="OSC_XI_GEOM=0";; *) ENV="";; esac
  env $ENV timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/xg_${v}_$rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/xg_${v}_$rep.json')); print('$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
done
