# A/B: warps per CTA of the level-0 ring up sweep (OSC_SUR_W 4 / 2 / 1) on cfg4 + parity subset
mkdir -p gpurun_out
for v in w2 w1; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "solve or nested or level_draws or cfg4" > gpurun_out/pytest_ab_$v.log 2>&1; echo "pytest $v $?"; tail -1 gpurun_out/pytest_ab_$v.log
done
for i in 1 2; do for v in base w2 w1; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_$i.json')); k=d['kernels_ms_profiled_step']
sel=['mg_smooth_up_r.L0@2048','mg_smooth_up_r.L0@1024']
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], [round(k.get(s,0),2) for s in sel], d['config']['mean_iters_fine'])"
done; done
