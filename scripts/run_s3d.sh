# CE twiddle prefetch + chunk-size A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "ce_ or level_draws or cfg4" > gpurun_out/pytest_s3d.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3d.log
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{}) or d.get('kernels_ms',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'ce_' in a})" $1; }
for mb in 80 160 400; do
  OSC_CE_CHUNK_MB=$mb timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ce_mb${mb}_c2.json 2>/dev/null; show gpurun_out/ce_mb${mb}_c2.json
  OSC_CE_CHUNK_MB=$mb timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ce_mb${mb}_c4.json 2>/dev/null; show gpurun_out/ce_mb${mb}_c4.json
done
CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
for k in ce_rows ce_cols; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_ce4_$k $CMD > gpurun_out/ncu_ce4_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_ce4_$k.ncu-rep 25 > gpurun_out/prof_ce4_$k.txt 2>&1
done
