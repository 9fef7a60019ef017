# ncu --set full of the level-0 up sweep and the coarse up sweep (2048^2 solve, batch 8), HEAD
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_s4.json 2>&1 || exit 1
for spec in "smooth_up_ring_kernel 2" "c_up_ring_kernel 10" "restrict_ring_kernel 2"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_s4_$1 $CMD > gpurun_out/ncu_s4_$1.log 2>&1
  tail -1 gpurun_out/ncu_s4_$1.log
done
