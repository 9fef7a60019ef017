# clock sampler started (and its NVML start-up finished) before the timed region: run-to-run spread
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s6d_$i.json 2> gpurun_out/s6d.err; echo "bench $?"
  python -c "
import json; d=json.load(open('gpurun_out/s6d_$i.json')); k=d['kernels_ms_profiled_step']
print(round(d['value'],1), round(d['e2e']['value'],1), d['ms_per_step'], round(sum(k.values()),1), d['clocks'])"
done
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s6d_c1.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s6d_c1.json')); print('c1', round(d['value']), round(d['e2e']['value']), d['clocks'])"
