bash scripts/ab_bench.sh dn4 dn5 dn6
python scripts/ab_compare.py gpurun_out/ab_dn4.json gpurun_out/ab_dn5.json gpurun_out/ab_dn6.json
OSC_LIB=$PWD/ab/dn6.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "solve_vs_oracle or galerkin_fewer" 2>&1 | tail -3
