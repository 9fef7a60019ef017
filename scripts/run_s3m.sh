# CE row pass: two row pairs per thread (default) vs one (OSC_CE_ROWS2=0); cols2 default
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{}) or d.get('kernels_ms',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'ce_' in a})" $1; }
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "ce_ or normals or level_draws_golden or host_xi" > gpurun_out/pytest_s3m.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_s3m.log
for rep in 1 2; do
for v in two one; do
  case $v in one) ENV="OSC_CE_ROWS2=0";; *) ENV="";; esac
  env $ENV timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2x_${v}_$rep.json 2>/dev/null; show gpurun_out/r2x_${v}_$rep.json
done
done
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2x_c4.json 2>/dev/null; show gpurun_out/r2x_c4.json
