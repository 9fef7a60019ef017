set -x
TAG=${1:-x}
python scripts/debug_fail.py > gpurun_out/dbg_fail_$TAG.log 2>&1; cat gpurun_out/dbg_fail_$TAG.log
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg3_$TAG.json 2> gpurun_out/cfg3_$TAG.err
python -c "import json; d=json.loads(open('gpurun_out/cfg3_$TAG.json').read()); print({k:(round(v['samples_per_s']),v.get('non_converged_sample_indices')) for k,v in d['per_level'].items()})"
python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg1_$TAG.json 2> gpurun_out/cfg1_$TAG.err
tail -n 2 gpurun_out/cfg1_$TAG.json | cut -c1-300
timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_$TAG.log
