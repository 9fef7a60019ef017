timeout 300 python scripts/ce_split.py > gpurun_out/r2g_ce_split.json 2>gpurun_out/r2g_ce.err; cat gpurun_out/r2g_ce_split.json; tail -3 gpurun_out/r2g_ce.err
timeout 900 python -m pytest tests -m gpu -q -x -rfE -p no:cacheprovider -k "ce_ or fields or golden or covariance or setup or smoothing or normals" > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2g_pytest.log
