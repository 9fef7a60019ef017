timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_v2.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_v2.log
timeout 600 python scripts/iters.py 64 256 2048 2>&1 | tail -8
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err; echo "bench exit $?"; cat gpurun_out/bench_v2.json | head -c 2500; tail -3 gpurun_out/bench_v2.err
