timeout 900 python -m pytest tests/test_gpu_setup.py tests/test_gpu_parity.py -q -rfE -p no:cacheprovider -k "setup or smoothing or level_create or osc1 or fields" > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2b_pytest.log
bash scripts/measure.sh r2b "cesplit ncu"
