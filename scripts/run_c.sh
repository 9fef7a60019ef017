# CE DIF vs Stockham (OSC_CE_DIF), fp32 p/z A/B, CE + solver parity
set -x
OSC_CE_DIF=0 timeout 300 python scripts/ce_split.py > gpurun_out/r2c_ce_split_stockham.json 2>gpurun_out/r2c_ce0.err; cat gpurun_out/r2c_ce_split_stockham.json
timeout 300 python scripts/ce_split.py > gpurun_out/r2c_ce_split_dif.json 2>gpurun_out/r2c_ce1.err; cat gpurun_out/r2c_ce_split_dif.json; tail -3 gpurun_out/r2c_ce1.err
timeout 1500 python -m pytest tests -m gpu -q -x -rfE -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2c_pytest.log
for c in 2; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2c_c$c.json 2> gpurun_out/r2c_c$c.err; python -c "
import json; d=json.load(open('gpurun_out/r2c_c$c.json')); print(d['value'], d['kernels_ms'])"; done
bash scripts/ab_bench.sh pz64 pz32
python scripts/ab_compare.py gpurun_out/ab_pz64.json gpurun_out/ab_pz32.json
