bash scripts/ab_bench.sh base z32 pz32
python scripts/ab_compare.py gpurun_out/ab_base.json gpurun_out/ab_z32.json gpurun_out/ab_pz32.json
