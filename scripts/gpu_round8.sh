set -x
TAG=${1:-x}
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg4_$TAG.json 2> gpurun_out/cfg4_$TAG.err
python -c "import json; d=json.loads(open('gpurun_out/cfg4_$TAG.json').read()); print(d['value'], d['roofline']['frac'], d['clocks'], list(d['kernels_ms_profiled_step'].items())[:10])"
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_$TAG.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4e_$TAG.json 2> gpurun_out/cfg4e_$TAG.err
python -c "import json; d=json.loads(open('gpurun_out/cfg4e_$TAG.json').read()); print(d['value'], d['e2e']['value'])"
