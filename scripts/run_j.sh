timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rfE -p no:cacheprovider -k "odd_coarsest or solve_vs_oracle or edge" > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2j_pytest.log
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_c2.json 2> gpurun_out/r2j_c2.err; python -c "
import json; d=json.load(open('gpurun_out/r2j_c2.json')); print(d['value'], d['resident_xi'], d['e2e'], d['kernels_ms'])"; tail -3 gpurun_out/r2j_c2.err
