#!/bin/bash
# GPU tests + benches for the Galerkin coarse-operator change
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gal_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gal_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/gal_cfg4.json 2> gpurun_out/gal_cfg4.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --coarse-op rediscretize > gpurun_out/gal_cfg4_redisc.json 2> gpurun_out/gal_cfg4_redisc.err
timeout 300 python bench.py --config 1 --no-cpu-baseline --no-e2e > gpurun_out/gal_cfg1.json 2>&1
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/gal_cfg3.json 2>&1
timeout 300 python bench.py --config 3 --mlmc > gpurun_out/gal_mlmc.json 2>&1
tail -3 gpurun_out/gal_tests.log
