mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s3p.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3p.log
for c in 4 3 1; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3p_c$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s3p_c$c.json')); print($c, round(d['value'],1), d['config'].get('mean_iters_fine'), d['clocks']['sm_mhz'])"; done
