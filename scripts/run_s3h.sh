mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s3h.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3h.log
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_s3h_c2.json 2> gpurun_out/bench_s3h_c2.err; echo "c2 exit $?"; head -c 1500 gpurun_out/bench_s3h_c2.json
