"""Turn an .ncu-rep into the markdown summary kept under profiles/ (headline counters of the first kernel + the ten
instructions that collect the most stall samples).  python tools/ncu_md.py <rep> <out.md> "<title>" "<command>" "<workload>" """
import csv, subprocess, sys
rep, out, title, cmd, work = sys.argv[1:6]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
keep = ("gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_active.avg")
lines = [f"# {title}", "", f"Command: `{cmd}`", f"Workload of the launch: {work}", "", f"Kernel: `{vals[hdr.index('Kernel Name')]}`", "",
         "| metric | value | unit |", "|---|---|---|"]
for h, u, v in zip(hdr, units, vals):
    if h in keep or ("issue_stalled" in h and h.endswith("per_issue_active.ratio") and "not_issued" not in h):
        lines.append(f"| {h} | {v} | {u} |")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
if len(srows) > 2:
    sh = srows[1]
    ia, isrc, iex, ismp = sh.index("Address"), sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in srows[2:]:
        try:
            data.append((int(r[ismp] or 0), r))
        except Exception:
            pass
    tot = sum(s for s, _ in data) or 1
    lines += ["", "Instructions with the most warp-stall samples (share of all samples of the kernel, top stall reasons):", "",
              "| share | SASS | executed | reasons |", "|---|---|---|---|"]
    for s, r in sorted(data, key=lambda x: -x[0])[:10]:
        st = {h[6:]: int(v) for h, v in zip(sh, r) if h.startswith("stall_") and "(" not in h and v not in ("", "0")}
        top = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        lines.append(f"| {100.0 * s / tot:.2f} % | `{r[isrc].strip()[:70]}` | {r[iex]} | {top} |")
open(out, "w").write("\n".join(lines) + "\n")
print(out)
