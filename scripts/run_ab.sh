# A/B of up-kernel ring depth / launch bounds (level stats on)
for v in r3b4 r4b3 r3b3 r5b2; do
  OSC_LEVEL_STATS=1 OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err; echo "$v exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); k=d['kernels_ms_profiled_step']; g=d['kernel_gbs']
print('$v value', round(d['value'],1), {n: (k[n], g.get(n)) for n in k if '@2048' in n and 'mg_up' in n})"
done
