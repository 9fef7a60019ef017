for c in 1; do
timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-e2e > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "cfg$c exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_cfg$c.json')); print(d['value'], d['ms_per_step'], d['config']['mean_iters_fine'], d['pipeline_roofline']['frac'], d['cpu_baseline']); print(d['kernels_ms'])"; tail -2 gpurun_out/bench_cfg$c.err
done
