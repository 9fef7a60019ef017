timeout 1500 python -m pytest tests -m gpu -q -x -rfE -p no:cacheprovider > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2l_pytest.log
timeout 300 python scripts/ce_split.py > gpurun_out/r2l_ce_split.json 2>gpurun_out/r2l_ce.err; cat gpurun_out/r2l_ce_split.json
timeout 2400 python scripts/cfg5_sweep.py > gpurun_out/r2l_cfg5.log 2>&1; echo "cfg5 rc=$?"; tail -30 gpurun_out/r2l_cfg5.log | cut -c1-400
