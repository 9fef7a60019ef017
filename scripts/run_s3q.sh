# CE intermediate with interleaved column pairs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "ce_ or level_draws or host_xi or smoothing" > gpurun_out/pytest_s3q.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_s3q.log
timeout 300 python scripts/ce_split.py 2>&1 | tail -1
for c in 2 4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3q_c$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s3q_c$c.json')); k=d.get('kernels_ms_profiled_step') or d.get('kernels_ms'); print($c, round(d['value'],1), d['clocks']['sm_mhz'], {a:b for a,b in k.items() if 'ce_' in a})"; done
