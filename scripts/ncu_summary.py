"""Summarise an ncu report: key throughput metrics + top stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active"]
units = rows[1] if len(rows) > 1 else []
for r in rows[2:]:
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:64s} {r[i][:60]} {units[i] if units else ''}")
    stalls = [(hdr[i], r[i]) for i in range(len(hdr)) if hdr[i].startswith("smsp__average_warp_latency_issue_stalled") or hdr[i].startswith("smsp__pcsamp_warps_issue_stalled")]
    vals = []
    for h, v in stalls:
        try:
            vals.append((float(v.replace(",", "")), h))
        except ValueError:
            pass
    for v, h in sorted(vals, reverse=True)[:8]:
        print(f"    stall {h:80s} {v}")
