#!/bin/bash
mkdir -p gpurun_out
OSC_LEVEL_STATS=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/lvl.json 2> gpurun_out/lvl.err
