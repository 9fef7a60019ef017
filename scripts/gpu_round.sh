# On the GPU box: GPU tests, smoke, and the bench lines; everything under gpurun_out/
set -x
TAG=${1:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
python bench.py --config 2 --batch 512 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c2_$TAG.json 2> gpurun_out/c2_$TAG.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4_$TAG.json 2> gpurun_out/cfg4_$TAG.err
tail -2 gpurun_out/*_$TAG.err
