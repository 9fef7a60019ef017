"""Per-source-line stall share of an ncu report: python scripts/ncu_lines.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ist = hdr.index("Warp Stall Sampling (All Samples)")
iie = hdr.index("Instructions Executed")
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
lines = [r for r in rows[hi + 1:] if len(r) > iie and r[0] not in ("",)]
tot = sum(f(r[ist]) for r in lines) or 1
toti = sum(f(r[iie]) for r in lines) or 1
for r in sorted(lines, key=lambda r: -f(r[ist]))[:n]:
    print(f"{100 * f(r[ist]) / tot:5.1f}% stall {100 * f(r[iie]) / toti:5.1f}% inst  L{r[0]}: {r[1].strip()[:100]}")
