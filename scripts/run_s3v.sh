mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "fused_setup or solve_vs_oracle or galerkin" > gpurun_out/pytest_s3v.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_s3v.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3v_c4.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s3v_c4.json')); k=d['kernels_ms_profiled_step']; print(round(d['value'],1), d['clocks']['sm_mhz'], {a:b for a,b in k.items() if 'setup' in a})"
