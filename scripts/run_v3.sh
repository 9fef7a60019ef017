timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_v13.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_v13.log
OSC_HARD_ITER_CAP=400 timeout 600 python scripts/iters.py 2048 2>&1 | tail -3
OSC_HARD_ITER_CAP=400 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_v13.json 2> gpurun_out/bench_v13.err; echo "bench exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_v13.json')); print(d['value'], d['config']['mean_iters_fine'], d['pipeline_roofline']['frac']); print(d['kernels_ms'])"; tail -3 gpurun_out/bench_v13.err
