# CE register-budget A/B (rows 3 or 2 CTAs/SM, cols 3) + full-chunk ncu of the CE kernels
mkdir -p gpurun_out
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{}) or d.get('kernels_ms',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'ce_' in a})" $1; }
for rep in 1 2; do
for v in base ce_r3 ce_r2 ce_c3; do
  case $v in base) LIBV=$PWD/paper_2306_13493_b200/libosc_b200.so;; *) LIBV=$PWD/ab/$v.so;; esac
  OSC_LIB=$LIBV timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mb_${v}_$rep.json 2>/dev/null; show gpurun_out/mb_${v}_$rep.json
done
done
CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 31 --no-cpu-baseline --no-e2e"
for k in ce_rows ce_cols; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/prof_ce6_$k $CMD > gpurun_out/ncu_ce6_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_ce6_$k.ncu-rep 25 > gpurun_out/prof_ce6_$k.txt 2>&1
done
