timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_v15.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_v15.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_v15.json 2> gpurun_out/bench_v15.err; echo "bench exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_v15.json')); print(d['value'], d['config']['mean_iters_fine'], d['roofline']); print(d['kernels_ms'])"; tail -3 gpurun_out/bench_v15.err
timeout 600 python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c2b.json 2> gpurun_out/bench_c2b.err; echo "c2 exit $?"; cat gpurun_out/bench_c2b.json; tail -3 gpurun_out/bench_c2b.err
