timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2u_cfg4_20steps.json 2> gpurun_out/r2u_cfg4_20steps.err; echo "bench rc=$?"
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2u_ref_20steps.json 2> gpurun_out/r2u_ref_20steps.err; echo "ref rc=$?"
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_c3.json 2> gpurun_out/r2u_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2u_c1.json 2> gpurun_out/r2u_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --config 3 --mlmc > gpurun_out/r2u_mlmc.json 2> gpurun_out/r2u_mlmc.err; echo "mlmc rc=$?"
timeout 2400 python scripts/cfg5_sweep.py --no-cpu > gpurun_out/r2u_cfg5.log 2> gpurun_out/r2u_cfg5.err; echo "cfg5 rc=$?"; cp gpurun_out/cfg5_sweep.json gpurun_out/r2u_cfg5_sweep.json
