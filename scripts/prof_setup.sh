CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
for spec in "galerkin_tile_kernel<true> 0" "galerkin_tile_kernel<false> 1"; do
  set -- $spec
  nm=$(echo $1 | tr -d '<>')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:galerkin_tile -s $2 -c 1 --kernel-name-base demangled -o gpurun_out/prof_s_$nm $CMD > gpurun_out/ncu_s_$nm.log 2>&1
  tail -1 gpurun_out/ncu_s_$nm.log
done
