# full GPU suite + CE chunk A/B at 1 GiB default + ncu of the CE kernels at a large chunk
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s3e.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3e.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{}) or d.get('kernels_ms',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'ce_' in a})" $1; }
for mb in 1024 3000; do
  OSC_CE_CHUNK_MB=$mb timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ce_mb${mb}_c2.json 2>/dev/null; show gpurun_out/ce_mb${mb}_c2.json
  OSC_CE_CHUNK_MB=$mb timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ce_mb${mb}_c4.json 2>/dev/null; show gpurun_out/ce_mb${mb}_c4.json
done
CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 32 --no-cpu-baseline --no-e2e"
for k in ce_rows ce_cols; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_ce5_$k $CMD > gpurun_out/ncu_ce5_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_ce5_$k.ncu-rep 25 > gpurun_out/prof_ce5_$k.txt 2>&1
done
