timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['e2e'])"; tail -2 gpurun_out/bench_e2e.err
