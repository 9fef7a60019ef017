# CE cols occupancy A/B (5 CTAs/SM at 48 regs vs 4 vs 3), carveout 100
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{}) or d.get('kernels_ms',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'ce_' in a})" $1; }
mkdir -p gpurun_out
for rep in 1 2; do
for v in base ce_c5 ce_c6 ce_c3; do
  case $v in base) LIBV=$PWD/paper_2306_13493_b200/libosc_b200.so;; *) LIBV=$PWD/ab/$v.so;; esac
  OSC_LIB=$LIBV timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/oc_${v}_$rep.json 2>/dev/null; show gpurun_out/oc_${v}_$rep.json
done
done
