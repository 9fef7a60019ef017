timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_e2e4.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_e2e4.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e4.json 2> gpurun_out/bench_e2e4.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_e2e4.json')); print(round(d['value'],1), d['e2e'], d['clocks'])"
