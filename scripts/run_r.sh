bash scripts/ab_bench.sh base cint
python scripts/ab_compare.py gpurun_out/ab_base.json gpurun_out/ab_cint.json
OSC_LIB=$PWD/ab/cint.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "solve or nested or level_draws or galerkin or streaming or device_loop or cfg4 or slot" 2>&1 | tail -4
