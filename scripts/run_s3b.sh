# fp64 peak; nested-iteration A/B (cfg4, cfg3, cfg1) after the 32-bit index fix; CE ncu captures
mkdir -p gpurun_out
./scripts/micro/fp64bench > gpurun_out/fp64bench.json 2>&1 || nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64b scripts/micro/fp64bench.cu && /tmp/fp64b > gpurun_out/fp64bench.json
cat gpurun_out/fp64bench.json
for rep in 1 2; do
for v in nested plain; do
  case $v in plain) ENV="OSC_NO_NESTED=1";; *) ENV="";; esac
  for c in 4 3 1; do
    env $ENV timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/nest_${v}_c${c}_$rep.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/nest_${v}_c${c}_$rep.json'))
k=d.get('kernels_ms_profiled_step',{})
print('$v c$c rep$rep', round(d['value'],1), d['ms_per_step'], d['config'].get('mean_iters_fine'), d['config'].get('mean_iters_coarse'), d['clocks']['sm_mhz'], 'init', k.get('pcg_init@2048', k.get('pcg_init@256')))"
  done
done
done
bash scripts/prof_ce.sh
for k in ce_rows ce_cols; do python scripts/ncu_summary.py gpurun_out/prof_ce2_$k.ncu-rep 25 > gpurun_out/prof_ce2_$k.txt 2>&1; done
