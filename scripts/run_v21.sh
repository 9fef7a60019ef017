#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/v22_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v22_tests.log
bash scripts/ab_bench.sh cur hybrid
tail -3 gpurun_out/v22_tests.log
