#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/v20_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v20_tests.log
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_v20.json 2>&1 || exit 1
for spec in "smooth_up_kernel 5" "update_down 2"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_v20_$1 $CMD > gpurun_out/ncu_v20_$1.log 2>&1
  tail -1 gpurun_out/ncu_v20_$1.log
done
tail -2 gpurun_out/v20_tests.log
