python scripts/ce_split.py --n4096; 
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2o_cfg4_20.json 2> gpurun_out/r2o.err; python -c "
import json; d=json.load(open('gpurun_out/r2o_cfg4_20.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks'])"
