set -x
TAG=${1:-x}
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_$TAG.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg4_$TAG.json 2> gpurun_out/cfg4_$TAG.err
python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg1_$TAG.json 2> gpurun_out/cfg1_$TAG.err
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg3_$TAG.json 2> gpurun_out/cfg3_$TAG.err
python bench.py --config 3 --mlmc --eps 1e-3 > gpurun_out/mlmc_$TAG.json 2> gpurun_out/mlmc_$TAG.err
tail -n 3 gpurun_out/*_$TAG.err
