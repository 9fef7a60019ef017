set -x
TAG=${1:-x}
timeout 900 python scripts/debug_cfg3_levels.py 1000000 > gpurun_out/dbg_cfg3_$TAG.log 2>&1
timeout 900 python scripts/debug_cfg3_levels.py 1000001 >> gpurun_out/dbg_cfg3_$TAG.log 2>&1
cat gpurun_out/dbg_cfg3_$TAG.log
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_$TAG.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4_$TAG.json 2> gpurun_out/cfg4_$TAG.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg4b_$TAG.json 2> gpurun_out/cfg4b_$TAG.err
python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg1_$TAG.json 2> gpurun_out/cfg1_$TAG.err
