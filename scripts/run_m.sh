timeout 900 python -m pytest tests/test_gpu_estimators.py -q -x -rfE -p no:cacheprovider > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2m_pytest.log
timeout 3000 python scripts/cfg5_sweep.py > gpurun_out/r2m_cfg5.log 2>&1; echo "cfg5 rc=$?"; python - <<'PY'
import json
d=json.load(open('gpurun_out/cfg5_sweep.json'))
for r in d['sweep']: print(r['lam'], r['eps'], r['variant'], round(r['wall_s'],2), r['n'], r['converged'], round(r['samples_per_s']))
for r in d['cpu_beside']: print('beside', r['lam'], r['eps'], r['variant'], round(r['gpu_wall_s'],3), round(r['cpu_wall_s'],2), round(r['speedup'],1), r['same_n'], r['n_cpu'])
PY
cp gpurun_out/cfg5_sweep.json gpurun_out/r2m_cfg5_sweep.json
