# self-contained nested start (one marching pass instead of init + nested)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "nested or level_draws or cfg4 or host_xi or slot or mlmc" > gpurun_out/pytest_s3t.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_s3t.log
for c in 4 3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3t_c$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s3t_c$c.json')); k=d.get('kernels_ms_profiled_step'); print($c, round(d['value'],1), d['config'].get('mean_iters_fine'), d['clocks']['sm_mhz'], {a:b for a,b in k.items() if 'init' in a})"; done
