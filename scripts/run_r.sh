timeout 2400 python -m pytest tests -m gpu -q -rfE -x -p no:cacheprovider > gpurun_out/r4c_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r4c_pytest_gpu.log
timeout 600 python scripts/level_breakdown.py 0,1,2,3 > gpurun_out/r4c_levels.json 2> gpurun_out/r4c_levels.err; echo "levels rc=$?"; tail -3 gpurun_out/r4c_levels.err
for T in 256 512 1024; do OSC_SMALL_T=$T timeout 600 python scripts/level_breakdown.py 0,1,2 > gpurun_out/r4c_levels_T$T.json 2>> gpurun_out/r4c_levels.err; done
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4c_c1.json 2> gpurun_out/r4c_c1.err; echo "c1 rc=$?"
