"""Print the headline counters of the first kernel in an .ncu-rep (issue rate, pipes, stalls, DRAM bytes)."""
import csv, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    print("##", vals[hdr.index("Kernel Name")][:100])
    for h, u, v in zip(hdr, units, vals):
        keep = h in ("gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                     "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
                     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
                     "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__warps_eligible.avg.per_cycle_active",
                     "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_active.avg")
        if keep or ("issue_stalled" in h and h.endswith("per_issue_active.ratio") and "not_issued" not in h):
            print(f"| {h} | {v} | {u} |")
