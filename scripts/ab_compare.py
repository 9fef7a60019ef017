"""Compare A/B bench lines: python scripts/ab_compare.py gpurun_out/ab_*.json"""
import json
import sys

rows = {}
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    rows[f] = d
keys = set()
for d in rows.values():
    keys |= set(d.get("kernels_ms", {}))
top = sorted(keys, key=lambda k: -max(d.get("kernels_ms", {}).get(k, 0) for d in rows.values()))[:14]
names = [f.split("/")[-1].replace(".json", "") for f in rows]
print(f"{'':30s}" + "".join(f"{n:>14s}" for n in names))
print(f"{'value':30s}" + "".join(f"{d['value']:14.2f}" for d in rows.values()))
print(f"{'iters f/c':30s}" + "".join(f"{d['config'].get('mean_iters_fine', 0):7.2f}/{(d['config'].get('mean_iters_coarse') or 0):6.2f}" for d in rows.values()))
for k in top:
    print(f"{k:30s}" + "".join(f"{d.get('kernels_ms', {}).get(k, 0) / d['steps']:14.2f}" for d in rows.values()))
for k in sorted(set().union(*[d.get("kernel_gbs", {}).keys() for d in rows.values()])):
    print(f"GB/s {k:25s}" + "".join(f"{d.get('kernel_gbs', {}).get(k, 0):14.0f}" for d in rows.values()))
