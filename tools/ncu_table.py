"""Per-kernel table from an .ncu-rep (time, issue %, warps active, DRAM bytes, hit rates)."""
import csv, io, subprocess, sys

M = ["gpu__time_duration.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
     "launch__registers_per_thread", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"]
SHORT = ["us", "issue%", "warps%", "dramR MB", "dramW MB", "winst M", "L1hit", "L2hit", "regs", "lsb", "bar", "membar", "lgthr"]
out = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}
idx = [h.index(m) if m in h else None for m in M]
print(f"{'kernel':24s}" + "".join(f"{s:>9s}" for s in SHORT))
for r in rows[2:]:
    name = r[h.index("Kernel Name")].replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:24]
    vals = []
    for m, i in zip(M, idx):
        v = float(r[i].replace(",", "")) if i is not None and r[i] not in ("", "n/a") else float("nan")
        if m.startswith("gpu__time"): v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(units[i], 1.0)
        if m.startswith("dram__bytes"): v *= SCALE.get(units[i], 1e-6)
        if m == "smsp__inst_executed.sum": v /= 1e6
        vals.append(v)
    print(f"{name:24s}" + "".join(f"{v:9.1f}" for v in vals))
