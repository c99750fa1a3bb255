"""Compact per-kernel table from an .ncu-rep (ncu -i ... --page raw --csv)."""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
     "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "launch__grid_size"]
short = ["us", "dram%", "dramMB", "warps%", "regs", "sm%", "winst", "l2hit", "lsb", "bar", "lgthr", "grid"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
print("kernel".ljust(34), " ".join(s.rjust(7) for s in short))
for r in rows[2:]:
    vals = []
    for m in M:
        v = r[ix[m]] if m in ix else ""
        try:
            f = float(v.replace(",", ""))
            if m == "gpu__time_duration.sum":
                f /= 1e3 if f > 1000 else 1
            if m == "dram__bytes_read.sum":
                f /= 1e6
            if m == "smsp__inst_executed.sum":
                f /= 1e6
            vals.append(f"{f:7.2f}")
        except ValueError:
            vals.append(v[:7].rjust(7))
    print(r[ix["Kernel Name"]][:34].ljust(34), " ".join(vals))
