bash scripts/ab_bench.sh base cdpf3 cdpf6
python scripts/ab_compare.py gpurun_out/ab_base.json gpurun_out/ab_cdpf3.json gpurun_out/ab_cdpf6.json
