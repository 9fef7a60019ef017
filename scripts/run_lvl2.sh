# setup P-stage split: targeted tests; level stats bench; CE kernels ncu at cfg4 (n = 4096)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fused_setup or galerkin_fewer or solve_vs_oracle or cfg4" > gpurun_out/pytest_lvl2.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_lvl2.log
OSC_LEVEL_STATS=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_lvl2.json 2> gpurun_out/bench_lvl2.err; echo "bench exit $?"
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
for spec in "ce_rows 1" "ce_cols 1"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_ce4_$1 $CMD > gpurun_out/ncu_ce4_$1.log 2>&1
  tail -1 gpurun_out/ncu_ce4_$1.log
done
