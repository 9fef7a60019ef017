timeout 900 python bench.py --config 3 --mlmc --eps 1e-3 > gpurun_out/mlmc_c3.json 2> gpurun_out/mlmc_c3.err; echo "exit $?"; cat gpurun_out/mlmc_c3.json; tail -5 gpurun_out/mlmc_c3.err
