timeout 2400 python -m pytest tests -m gpu -q -rfE -x -p no:cacheprovider > gpurun_out/r4i_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r4i_pytest_gpu.log
for c in 1 3; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r4i_c$c.json 2> gpurun_out/r4i_c$c.err; echo "c$c rc=$?"
done
timeout 900 python bench.py --config 3 --mlmc > gpurun_out/r4i_mlmc.json 2> gpurun_out/r4i_mlmc.err; echo "mlmc rc=$?"
timeout 600 python scripts/level_breakdown.py 2 > gpurun_out/r4i_levels.json 2> gpurun_out/r4i_levels.err
timeout 600 python scripts/level_breakdown.py 2 >> gpurun_out/r4i_levels.json 2>> gpurun_out/r4i_levels.err
