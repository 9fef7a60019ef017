bash scripts/ab_bench.sh base rcp1
python scripts/ab_compare.py gpurun_out/ab_base.json gpurun_out/ab_rcp1.json
OSC_LIB=$PWD/ab/rcp1.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "solve or nested or level_draws or galerkin or streaming or device_loop" 2>&1 | tail -4
