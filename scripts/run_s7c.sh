# A/B: coarse up-sweep ring depth (OSC_UP_RING 3 / 4 / 5) with one-warp CTAs, cfg4
mkdir -p gpurun_out
OSC_LIB=$PWD/ab/ur5.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "solve or nested or cfg4" > gpurun_out/pytest_ab_ur5.log 2>&1; echo "pytest ur5 $?"; tail -1 gpurun_out/pytest_ab_ur5.log
for i in 1 2; do for v in head ur4 ur5; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_$i.json')); k=d['kernels_ms_profiled_step']
sel=['mg_up.Lc@2048','mg_up.Lc@1024']
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], [round(k.get(s,0),2) for s in sel], round(sum(k.values()),1))"
done; done
