# ncu --set full of the level-0 kernels of the one-reduction PCG (2048^2 solve, batch 8)
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_l0.json 2>&1 || exit 1
for spec in "smooth_up_r_kernel 2" "restrict_r_kernel 2" "pcg_update_cg_kernel 2"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_l0_$1 $CMD > gpurun_out/ncu_l0_$1.log 2>&1
  tail -1 gpurun_out/ncu_l0_$1.log
done
