set -x
TAG=${1:-x}
timeout 900 python scripts/debug_cfg3_levels.py 1000000 > gpurun_out/dbg_cfg3_$TAG.log 2>&1
cat gpurun_out/dbg_cfg3_$TAG.log
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg3_$TAG.json 2> gpurun_out/cfg3_$TAG.err
tail -n 5 gpurun_out/cfg3_$TAG.err
python -c "import json; d=json.loads(open('gpurun_out/cfg3_$TAG.json').read()); print(json.dumps(d['per_level'], indent=1))"
