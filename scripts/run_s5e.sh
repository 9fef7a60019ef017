# A/B: one-warp CTAs for the ring sweeps (smooth_up / restrict / coarse down / coarse up) on cfg4 + parity subset
mkdir -p gpurun_out
OSC_LIB=$PWD/ab/all1.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "solve or nested or level_draws or cfg4 or galerkin" > gpurun_out/pytest_ab_all1.log 2>&1; echo "pytest all1 $?"; tail -1 gpurun_out/pytest_ab_all1.log
for i in 1 2; do for v in base sur1 sur1rr1 all1; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_$i.json')); k=d['kernels_ms_profiled_step']
sel=['mg_smooth_up_r.L0@2048','mg_restrict_r.L0@2048','mg_up.Lc@2048','mg_down.Lc@2048','mg_smooth_up_r.L0@1024','mg_restrict_r.L0@1024','mg_up.Lc@1024','mg_down.Lc@1024']
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], [round(k.get(s,0),2) for s in sel], round(sum(k.values()),1))"
done; done
