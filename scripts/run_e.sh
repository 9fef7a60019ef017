timeout 300 python scripts/ce_split.py > gpurun_out/r2e_ce_split.json 2>gpurun_out/r2e_ce.err; cat gpurun_out/r2e_ce_split.json; tail -3 gpurun_out/r2e_ce.err
timeout 900 python -m pytest tests -m gpu -q -x -rfE -p no:cacheprovider -k "ce_ or fields or golden or covariance or setup or smoothing or normals" > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2e_pytest.log
for m in philox xi; do
  s=0; [ $m = xi ] && s=10
  timeout 600 ncu --set full --clock-control none -k regex:ce_ -s $s -c 2 -o gpurun_out/r2e_ce_$m python scripts/ce_split.py > gpurun_out/r2e_ncu_$m.log 2>&1
  python scripts/ncu_stalls.py gpurun_out/r2e_ce_$m.ncu-rep > gpurun_out/r2e_ce_${m}_stalls.txt 2>&1
  ncu -i gpurun_out/r2e_ce_$m.ncu-rep --page raw --csv > gpurun_out/r2e_ce_${m}_raw.csv 2>/dev/null
  rm -f gpurun_out/r2e_ce_$m.ncu-rep
  cat gpurun_out/r2e_ce_${m}_stalls.txt
done
