"""Summarise an ncu report: stalls, DRAM bytes, occupancy (run here, no GPU)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("kernel:", d.get("Kernel Name", "")[:80])
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for h, v in d.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v}
    tot = sum(stalls.values()) or 1
    print("  stalls:", ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]))
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
              "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__shared_mem_per_block_dynamic",
              "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active"):
        print(f"  {k} = {d.get(k)}")
