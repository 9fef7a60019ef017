set -x
TAG=${1:-x}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rfE -p no:cacheprovider -k "xi or prefetch or chunk" > gpurun_out/pytest_xi_$TAG.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_xi_$TAG.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4e_$TAG.json 2> gpurun_out/cfg4e_$TAG.err
python -c "import json; d=json.loads(open('gpurun_out/cfg4e_$TAG.json').read()); print(d['value'], d['e2e'])"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4e10_$TAG.json 2> gpurun_out/cfg4e10_$TAG.err
python -c "import json; d=json.loads(open('gpurun_out/cfg4e10_$TAG.json').read()); print(d['value'], d['e2e']['value'])"
