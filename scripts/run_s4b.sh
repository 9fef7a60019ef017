# e2e host-ξ chunk ramp A/B on cfg 4 (OSC_XI_FIRST_DIV=0: the old uniform 4 chunks)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "host_xi_chunks" > gpurun_out/pytest_s4b.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_s4b.log
for v in "" "OSC_XI_FIRST_DIV=0" "OSC_XI_RAMP=1.35" "OSC_XI_FIRST_DIV=32"; do
  env $v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4b.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s4b.json')); print('$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['h2d_gbs'],1), d['clocks']['sm_mhz'])"
done
# cfg1 / MLMC regression check against the 4b2387b build (ab/old_tree)
for i in 1 2; do
  timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4b_c1_new.json 2>/dev/null
  (cd ab/old_tree && timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline > ../../gpurun_out/s4b_c1_old.json 2>/dev/null)
  python -c "
import json
for t in ['new','old']:
  d=json.load(open(f'gpurun_out/s4b_c1_{t}.json')); print('c1', t, round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"
done
timeout 600 python bench.py --config 3 --mlmc > gpurun_out/s4b_mlmc_new.json 2>/dev/null
(cd ab/old_tree && timeout 600 python bench.py --config 3 --mlmc > ../../gpurun_out/s4b_mlmc_old.json 2>/dev/null)
python -c "
import json
for t in ['new','old']:
  d=json.load(open(f'gpurun_out/s4b_mlmc_{t}.json')); print('mlmc', t, d['wall_s'], [l['wall_per_sample_s'] for l in d['levels']])"
