# CE intermediate interleave width A/B (2 / 4 / 8 columns per q1 run)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "ce_ or level_draws_golden or host_xi" > gpurun_out/pytest_s3r.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_s3r.log
for v in il4 il2 il8 il4; do case $v in il4) LIBV=$PWD/paper_2306_13493_b200/libosc_b200.so;; *) LIBV=$PWD/ab/$v.so;; esac; echo $v; OSC_LIB=$LIBV timeout 300 python scripts/ce_split.py 2>&1 | tail -1; done
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3r_c2.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s3r_c2.json')); print(round(d['value'],1), d['kernels_ms'])"
