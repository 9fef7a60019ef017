# CE compile-time-n kernels + row-marching PCG init: GPU suite, A/B benches, fp64 peak, CE ncu
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/fp64bench scripts/micro/fp64bench.cu && ./gpurun_out/fp64bench > gpurun_out/fp64bench.json; cat gpurun_out/fp64bench.json
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s3c.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3c.log
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('mean_iters_fine'), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'ce_' in a or 'init' in a})" $1; }
for rep in 1 2; do
for v in new legacy; do
  case $v in legacy) ENV="OSC_CE_LEGACY=1";; *) ENV="";; esac
  env $ENV timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ce_${v}_c2_$rep.json 2>/dev/null; show gpurun_out/ce_${v}_c2_$rep.json
  env $ENV timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ce_${v}_c4_$rep.json 2>/dev/null; show gpurun_out/ce_${v}_c4_$rep.json
done
done
for v in nested plain; do
  case $v in plain) ENV="OSC_NO_NESTED=1";; *) ENV="";; esac
  env $ENV timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/n_${v}_c3.json 2>/dev/null; show gpurun_out/n_${v}_c3.json
  env $ENV timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/n_${v}_c4.json 2>/dev/null; show gpurun_out/n_${v}_c4.json
done
CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
for k in ce_rows ce_cols; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_ce3_$k $CMD > gpurun_out/ncu_ce3_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_ce3_$k.ncu-rep 25 > gpurun_out/prof_ce3_$k.txt 2>&1
done
