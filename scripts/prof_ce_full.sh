set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config 2 --batch 256 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c2_base.json 2> gpurun_out/c2_base.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ce_ -c 2 -o gpurun_out/ce_full python bench.py --config 2 --batch 32 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ce_ncu.log 2>&1
ls -la gpurun_out
