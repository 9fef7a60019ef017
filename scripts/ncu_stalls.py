"""Per kernel of an ncu report: warp-stall reasons (pc sampling), issue utilisation, opcode mix."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:70], r[hdr.index("Grid Size")], r[hdr.index("gpu__time_duration.sum")], "us")
    items = []
    for i, h in enumerate(hdr):
        if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
            try:
                items.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in items) or 1
    print("  stalls: " + ", ".join(f"{h} {v / tot * 100:.1f}%" for v, h in sorted(items, reverse=True)[:9]))
    for h in ["smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
              "smsp__warps_eligible.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
              "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
              "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
              "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum",
              "smsp__inst_executed_op_global_ld.sum", "smsp__inst_executed_op_global_st.sum",
              "smsp__inst_executed_op_ldgsts.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "lts__t_sectors.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
              "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_barriers"]:
        if h in hdr:
            print(f"  {h}: {r[hdr.index(h)]} {rows[1][hdr.index(h)]}")
    ops = []
    for i, h in enumerate(hdr):
        if h.startswith("sass__inst_executed_per_opcode"):
            ops.append((h, r[i]))
    for h, v in ops[:2]:
        print(f"  {h}: {v[:600]}")
