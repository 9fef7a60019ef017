# round-end style measurement set on the current code
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['e2e'], d['roofline']['kernel'], d['roofline']['frac'], d['pipeline_roofline']['frac'], d['cpu_baseline'], d['gpu_launches'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err; echo "ref exit $?"; cat gpurun_out/bench_final_ref.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_final_torchrun.json 2> gpurun_out/bench_final_torchrun.err; echo "torchrun exit $?"; head -c 300 gpurun_out/bench_final_torchrun.json; echo
for c in 1 2 3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_final_c$c.json 2> gpurun_out/bench_final_c$c.err; echo "c$c exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_final_c$c.json')); print(d['value'], (d.get('e2e') or {}).get('value'), d['pipeline_roofline']['frac'], (d.get('cpu_baseline') or {}).get('value'), d['roofline'].get('kernel'), d['roofline'].get('frac'))"
done
timeout 900 python bench.py --config 3 --mlmc > gpurun_out/bench_final_mlmc.json 2> gpurun_out/bench_final_mlmc.err; echo "mlmc exit $?"; head -c 600 gpurun_out/bench_final_mlmc.json; echo
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch_final.log 2>&1; echo "ncu launches exit $?"
