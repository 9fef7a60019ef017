CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
for spec in "c_up_ring_kernel 60 10" "c_down_ring_kernel 60 10"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none -k regex:$1 -s $2 -c $3 -o gpurun_out/r2q_$1 $CMD > gpurun_out/r2q_ncu_$1.log 2>&1
  python scripts/ncu_stalls.py gpurun_out/r2q_$1.ncu-rep > gpurun_out/r2q_$1_stalls.txt 2>&1
  rm -f gpurun_out/r2q_$1.ncu-rep
done
grep -A12 "(18, 17, 8)\|(5, 17, 8)" gpurun_out/r2q_c_up_ring_kernel_stalls.txt | head -30
grep -A12 "(5, 17, 8)\|(5, 33, 8)" gpurun_out/r2q_c_down_ring_kernel_stalls.txt | head -30
grep "^==" gpurun_out/r2q_c_down_ring_kernel_stalls.txt
