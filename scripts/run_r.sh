bash scripts/ab_bench.sh base c1 c2
python scripts/ab_compare.py gpurun_out/ab_base.json gpurun_out/ab_c1.json gpurun_out/ab_c2.json
