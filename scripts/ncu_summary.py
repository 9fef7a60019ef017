"""Summarise an ncu report: key metrics + top stall lines (source page)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ['Kernel Name', 'Grid Size', 'Block Size', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'lts__t_sectors.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'launch__occupancy_limit_shared_mem',
        'launch__registers_per_thread', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
for r in rows[2:]:
    for w in want:
        if w in hdr:
            print(f"  {w}: {r[hdr.index(w)]} {rows[1][hdr.index(w)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
if hi:
    hdr = rows[hi[0]]
    i_src = hdr.index('Source'); i_st = hdr.index('Warp Stall Sampling (All Samples)'); i_ie = hdr.index('Instructions Executed')
    def f(x):
        try: return float(x)
        except: return 0.0
    data = [r for r in rows[hi[0] + 1:] if len(r) > i_ie and r[0] != 'Address']
    tot = sum(f(r[i_st]) for r in data) or 1; tot_i = sum(f(r[i_ie]) for r in data) or 1
    print(f"  stall samples {tot:.0f}, warp instr {tot_i:.0f}")
    agg = {}
    for r in data:
        k = r[i_src].strip()[:90]
        a = agg.setdefault(k, [0, 0]); a[0] += f(r[i_st]); a[1] += f(r[i_ie])
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
        print(f"  {v[0]/tot*100:5.1f}% stall {v[1]/tot_i*100:5.1f}% instr | {k}")
