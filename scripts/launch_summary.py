"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time share per kernel."""
import csv, sys, collections, re
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    name = re.sub(r"\(.*", "", r[4]).replace("void ", "").replace("unnamed>::", "").replace("osc::", "")
    a = agg[name]; a[0] += 1; a[1] += float(r[-1])
tot = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches, {tot/1e6:.3f} ms total (ncu: cold-cache, serialised)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {v[1]/tot*100:5.1f}%  {v[1]/1e6:9.3f} ms  {v[0]:5d} launches  {k}")
