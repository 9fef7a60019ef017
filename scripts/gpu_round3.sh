set -x
TAG=${1:-x}
timeout 600 python scripts/debug_cfg3_levels.py > gpurun_out/dbg_cfg3_$TAG.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_$TAG.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4_$TAG.json 2> gpurun_out/cfg4_$TAG.err
cat gpurun_out/dbg_cfg3_$TAG.log
