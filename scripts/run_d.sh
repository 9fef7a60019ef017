# stall breakdown of the CE passes: Stockham vs DIF, device Philox vs resident xi
for dif in 0 1; do
  for spec in "philox 0" "xi 10"; do
    set -- $spec
    OSC_CE_DIF=$dif timeout 600 ncu --set full --clock-control none -k regex:ce_ -s $2 -c 2 -o gpurun_out/r2d_ce_dif${dif}_$1 python scripts/ce_split.py > gpurun_out/r2d_ncu_${dif}_$1.log 2>&1
    python scripts/ncu_stalls.py gpurun_out/r2d_ce_dif${dif}_$1.ncu-rep > gpurun_out/r2d_ce_dif${dif}_$1_stalls.txt 2>&1
    rm -f gpurun_out/r2d_ce_dif${dif}_$1.ncu-rep
    cat gpurun_out/r2d_ce_dif${dif}_$1_stalls.txt
  done
done
