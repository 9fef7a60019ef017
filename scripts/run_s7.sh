# round-end measurement set on HEAD (one-warp ring CTAs, clock sampler fix): full GPU suite, smoke, every bench
# workload, launch list, ncu --set full of the 2048^2 level-0 kernels
mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s7.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_s7.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/s7_cfg4.json 2> gpurun_out/s7_cfg4.err; echo "bench exit $?"
python -c "
import json; d=json.load(open('gpurun_out/s7_cfg4.json')); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['pipeline_roofline']['frac'], d['cpu_baseline'], d['gpu_launches'], d['clocks'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s7_ref.json 2> gpurun_out/s7_ref.err; echo "ref exit $?"; cat gpurun_out/s7_ref.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/s7_torchrun.json 2> gpurun_out/s7_torchrun.err; echo "torchrun exit $?"; head -c 300 gpurun_out/s7_torchrun.json; echo
for c in 1 2 3; do
  st=5; [ $c = 1 ] && st=30
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/s7_c$c.json 2> gpurun_out/s7_c$c.err; echo "c$c exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/s7_c$c.json')); print(d['value'], (d.get('e2e') or {}).get('value'), d['pipeline_roofline']['frac'], (d.get('cpu_baseline') or {}).get('value'), d['roofline'].get('kernel'), d['roofline'].get('frac'))"
done
timeout 900 python bench.py --config 3 --mlmc > gpurun_out/s7_mlmc.json 2> gpurun_out/s7_mlmc.err; echo "mlmc exit $?"; head -c 400 gpurun_out/s7_mlmc.json; echo
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/s7_launches.csv $CMD > gpurun_out/s7_ncu_launch.log 2>&1; echo "ncu launches exit $?"
for spec in "pcg_update_cg_kernel 20" "smooth_up_ring_kernel 20"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_s7_$1 $CMD > gpurun_out/ncu_s7_$1.log 2>&1
  tail -1 gpurun_out/ncu_s7_$1.log
done
