for m in 2048; do OSC_HARD_ITER_CAP=300 timeout 120 python scripts/diag.py $m 1; echo "exit $?"; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_v2.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_v2.log
OSC_HARD_ITER_CAP=400 timeout 600 python scripts/iters.py 256 1024 2048 2>&1 | tail -8
OSC_HARD_ITER_CAP=400 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err; echo "bench exit $?"; cat gpurun_out/bench_v2.json | head -c 3000; tail -3 gpurun_out/bench_v2.err
