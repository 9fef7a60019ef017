timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_v17.json 2> gpurun_out/bench_v17.err; echo "bench exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_v17.json')); print(d['value'], d['config']['mean_iters_fine'], d['config']['mean_iters_coarse']); print(d['kernels_ms'])"; tail -2 gpurun_out/bench_v17.err
timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err; echo "c3 exit $?"; python -c "
import json; d=json.load(open('gpurun_out/bench_c3b.json')); print(d['value'], d['config']['mean_iters_fine'], d['pipeline_roofline']['frac']); print(d['kernels_ms'])"
