timeout 300 python scripts/ce_split.py > gpurun_out/r2k_ce_split.json 2>gpurun_out/r2k_ce.err; cat gpurun_out/r2k_ce_split.json; tail -3 gpurun_out/r2k_ce.err
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_c2.json 2> gpurun_out/r2k_c2.err; python -c "
import json; d=json.load(open('gpurun_out/r2k_c2.json')); print(d['value'], d['resident_xi'], d['kernels_ms'])"; tail -3 gpurun_out/r2k_c2.err
timeout 900 python -m pytest tests -m gpu -q -x -rfE -p no:cacheprovider -k "ce_ or fields or golden or covariance or setup or smoothing or normals" > gpurun_out/r2k_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2k_pytest.log
