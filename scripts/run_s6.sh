# one-warp ring CTAs as the default: full GPU suite, smoke, default bench, CD_W=2 A/B
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s6.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_s6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/s6_cfg4.json 2> gpurun_out/s6_cfg4.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/s6_cfg4.json')); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['pipeline_roofline']['frac'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
for i in 1 2; do for v in head cd2; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_$i.json')); k=d['kernels_ms_profiled_step']
sel=['mg_down.Lc@2048','mg_down.Lc@1024']
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], [round(k.get(s,0),2) for s in sel], round(sum(k.values()),1))"
done; done
