# ramp (1.35, ≥ 256 MB gate) confirmation: host-ξ parity incl. the forced ramp, cfg4 e2e x2 vs uniform, cfg1 e2e; MLMC new/old x2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "host_xi_chunks" > gpurun_out/pytest_s4c.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_s4c.log
for i in 1 2; do
for v in "" "OSC_XI_FIRST_DIV=0"; do
  env $v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4c.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s4c.json')); print('c4 $v', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['value']/d['value'],3), d['clocks']['sm_mhz'])"
done; done
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4c_c1.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/s4c_c1.json')); print('c1', round(d['value']), round(d['e2e']['value']))"
for i in 1 2; do
timeout 600 python bench.py --config 3 --mlmc > gpurun_out/s4c_mlmc_new.json 2>/dev/null
(cd ab/old_tree && timeout 600 python bench.py --config 3 --mlmc > ../../gpurun_out/s4c_mlmc_old.json 2>/dev/null)
python -c "
import json
for t in ['new','old']:
  d=json.load(open(f'gpurun_out/s4c_mlmc_{t}.json')); print('mlmc', t, d['wall_s'], [round(l['wall_per_sample_s']*1e6,2) for l in d['levels']])"
done
