# tests + bench cfg4/cfg3 + CE ncu (instruction counts for the ceiling)
set -x
TAG=${1:-x}
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_$TAG.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4_$TAG.json 2> gpurun_out/cfg4_$TAG.err
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg3_$TAG.json 2> gpurun_out/cfg3_$TAG.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ce_ -c 2 -o gpurun_out/ce_full_$TAG python bench.py --config 2 --batch 32 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ce_ncu_$TAG.log 2>&1
tail -3 gpurun_out/*_$TAG.err
