bash scripts/ab_bench.sh base margin
python scripts/ab_compare.py gpurun_out/ab_base.json gpurun_out/ab_margin.json
python - <<'PY'
import json
for v in ('base','margin'):
    d=json.load(open(f'gpurun_out/ab_{v}.json')); k=d['kernels_ms_profiled_step']
    print(v, {n:t for n,t in k.items() if 'setup' in n})
PY
OSC_LIB=$PWD/ab/margin.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "solve or nested or level_draws or galerkin or streaming or device_loop or cfg4" 2>&1 | tail -4
