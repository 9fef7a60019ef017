# CE column pass: two columns per thread (OSC_CE_COLS2=1) vs one
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{}) or d.get('kernels_ms',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'ce_' in a})" $1; }
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "ce_fields" > gpurun_out/pytest_s3l_a.log 2>&1; echo "pytest base $?"
OSC_CE_COLS2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "ce_fields" > gpurun_out/pytest_s3l_b.log 2>&1; echo "pytest cols2 $?"; tail -3 gpurun_out/pytest_s3l_b.log
for rep in 1 2; do
for v in one two; do
  case $v in two) ENV="OSC_CE_COLS2=1";; *) ENV="";; esac
  env $ENV timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2x_${v}_$rep.json 2>/dev/null; show gpurun_out/c2x_${v}_$rep.json
done
done
env OSC_CE_COLS2=1 timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4x_two.json 2>/dev/null; show gpurun_out/c4x_two.json
