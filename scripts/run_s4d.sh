# cross-call xi prefetch: parity tests, then e2e on cfg4 (x2), cfg1, cfg3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "host_xi_chunks or xi_prefetch" > gpurun_out/pytest_s4d.log 2>&1; echo "pytest $?"; tail -15 gpurun_out/pytest_s4d.log
for i in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s4d_c4_$i.json 2>gpurun_out/s4d_c4.err; echo "bench $?"; tail -3 gpurun_out/s4d_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/s4d_c4_$i.json')); print('c4', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['value']/d['value'],3), d['e2e']['steps'], d['clocks']['sm_mhz'])"
done
for c in 1 3; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4d_c$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/s4d_c$c.json')); print('c$c', round(d['value']), round(d['e2e']['value']))"
done
