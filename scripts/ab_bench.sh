#!/bin/bash
# A/B: cfg4 bench per library variant in ab/ (OSC_LIB override), kernel bandwidths summarised
mkdir -p gpurun_out
for v in "$@"; do
  OSC_LIB=$PWD/ab/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
done
