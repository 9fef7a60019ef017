for v in cx2 cx4 cx8; do
  OSC_LIB=$PWD/ab/$v.so timeout 300 python scripts/ce_split.py > gpurun_out/r2h_ce_split_$v.json 2>gpurun_out/r2h_$v.err; echo $v; cat gpurun_out/r2h_ce_split_$v.json; tail -2 gpurun_out/r2h_$v.err
done
OSC_LIB=$PWD/ab/cx8.so timeout 900 python -m pytest tests -m gpu -q -x -rfE -p no:cacheprovider -k "ce_ or fields or golden or covariance or setup or smoothing" > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2h_pytest.log
