# A/B: register budget of the level-0 ring restriction (one-warp, 12 CTAs/SM) and the coarse down sweep (3 CTAs/SM)
mkdir -p gpurun_out
for i in 1 2; do for v in head rrm3 cdm3; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_$i.json')); k=d['kernels_ms_profiled_step']
sel=['mg_restrict_r.L0@2048','mg_restrict_r.L0@1024','mg_down.Lc@2048','mg_down.Lc@1024']
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], [round(k.get(s,0),2) for s in sel], round(sum(k.values()),1))"
done; done
