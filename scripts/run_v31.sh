#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v32_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v32_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v32_cfg4.json 2> gpurun_out/v32_cfg4.err
OSC_SIMPLE_COARSE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v32_cfg4_simple.json 2> gpurun_out/v32_cfg4_simple.err
tail -5 gpurun_out/v32_tests.log
