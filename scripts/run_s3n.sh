mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s3n.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s3n.log
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/bench_s3n_c2.json 2> gpurun_out/bench_s3n_c2.err; echo "c2 exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_s3n_c2.json')); print(d['value'], d['compute_roofline']['frac'], d['pipeline_roofline']['frac'], d['kernels_ms'])"
CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 31 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ce_cols -s 0 -c 1 -o gpurun_out/prof_ce7_ce_cols $CMD > gpurun_out/ncu_ce7_ce_cols.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_ce7_ce_cols.ncu-rep 25 > gpurun_out/prof_ce7_ce_cols.txt 2>&1
