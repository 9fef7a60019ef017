# ncu --set full of the CE kernels at config 2 (n = 2048, batch 8)
CMD="python bench.py --config 2 --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_ce.json 2>&1 || exit 1
for k in ce_rows ce_cols; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_ce2_$k $CMD > gpurun_out/ncu_ce2_$k.log 2>&1
  tail -1 gpurun_out/ncu_ce2_$k.log
done
