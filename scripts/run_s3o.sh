# rows per warp (64 at m >= 1024) and coarse rows per warp for the level-0 restriction (32 at mc >= 512)
show() { python -c "
import json,sys; d=json.load(open(sys.argv[1])); k=d.get('kernels_ms_profiled_step',{})
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('mean_iters_fine'), d['clocks']['sm_mhz'], {a: round(b,2) for a,b in k.items() if 'L0@2048' in a or 'pcg_update@2048' in a})" $1; }
mkdir -p gpurun_out
for rep in 1 2; do
for v in base rpw3 lyc32 both; do
  case $v in base) LIBV=$PWD/paper_2306_13493_b200/libosc_b200.so;; *) LIBV=$PWD/ab/$v.so;; esac
  OSC_LIB=$LIBV timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ly_${v}_$rep.json 2>/dev/null; show gpurun_out/ly_${v}_$rep.json
done
done
