timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "ce_ or golden or draws or normals or smoothing" 2>&1 | tail -2
timeout 600 python bench.py --config 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2c.json 2> gpurun_out/bench_c2c.err; echo "c2 exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_c2c.json')); print(d['value'], d['pipeline_roofline']['frac'], d['kernels_ms'])"; tail -2 gpurun_out/bench_c2c.err
