# round re-entry check: GPU parity suite, smoke, full default bench (value + e2e + cpu baseline), reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_state.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_state.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_state.json 2> gpurun_out/bench_state.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_state.json')); print(d['value'], d['e2e'], d['roofline'], d['pipeline_roofline']['frac'], d['cpu_baseline'], d['gpu_launches'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"; cat gpurun_out/bench_ref.json
