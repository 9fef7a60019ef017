# nested-iteration marching init: parity tests + A/B (march / simple / off) on cfg4 and cfg3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "nested or level_draws or cfg4 or slot or mlmc" > gpurun_out/pytest_s3g.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3g.log
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{}) or d.get('kernels_ms',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('mean_iters_fine'), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'init' in a})" $1; }
for rep in 1; do
for v in march simple; do
  case $v in simple) ENV="OSC_NESTED_SIMPLE=1";; off) ENV="OSC_NO_NESTED=1";; *) ENV="";; esac
  for c in 4 3; do
    env $ENV timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ns_${v}_c${c}_$rep.json 2>/dev/null; show gpurun_out/ns_${v}_c${c}_$rep.json
  done
done
done
