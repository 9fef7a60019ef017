for v in default nograph; do
  if [ $v = nograph ]; then export OSC_LIB=$PWD/ab/nograph.so; fi
  python scripts/cfg5_sweep.py 1e-2,1e-3 --no-cpu > gpurun_out/r2n_cfg5_$v.log 2>&1; echo "$v rc=$?"
  python - <<'PY'
import json
d=json.load(open('gpurun_out/cfg5_sweep.json'))
for r in d['sweep']: print(r['lam'], r['eps'], r['variant'], round(r['wall_s'],2), r['n'])
PY
done
