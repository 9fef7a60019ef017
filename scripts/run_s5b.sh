# A/B: level-0 rows per warp (OSC_RPW 4/5) and level-0 restriction coarse rows (OSC_LYC_BIG 48) on cfg4
mkdir -p gpurun_out
for i in 1 2; do for v in base rpw4 rpw5 lyc48; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_$i.json')); k=d['kernels_ms_profiled_step']
sel=['pcg_update@2048','mg_smooth_up_r.L0@2048','mg_restrict_r.L0@2048','pcg_update@1024','mg_smooth_up_r.L0@1024','mg_restrict_r.L0@1024']
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], [round(k.get(s,0),2) for s in sel], round(sum(k.get(s,0) for s in sel),2))"
done; done
