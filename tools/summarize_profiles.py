"""Turn the gpurun_out/ artefacts of tools/profile_round.sh into committed summaries in profiles/."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                d[k] = r[h.index(k)] + (" " + units[h.index(k)] if units[h.index(k)] else "")
        st = [(float(r[i]), x) for i, x in enumerate(h) if x.startswith("smsp__average_warps_issue_stalled")
              and x.endswith("_per_issue_active.ratio") and r[i] not in ("", "0")]
        d["top_stalls"] = {x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: v
                           for v, x in sorted(st, reverse=True)[:6]}
        res.append(d)
    return res


def main():
    summary = {}
    lines = []
    for cfg in ("C2", "C3", "G2"):
        rep = os.path.join(OUT, f"{TAG}_k_cast_{cfg}.ncu-rep")
        if os.path.exists(rep):
            for d in raw(rep):
                lines.append(f"## {cfg} {d['kernel']}")
                lines += [f"  {k:70s} {v}" for k, v in d.items() if k not in ("kernel", "top_stalls")]
                lines.append(f"  top stalls (warps per issued instruction): {d['top_stalls']}")
                rd = float(d["dram__bytes_read.sum"].split()[0]) * (1e6 if "Mbyte" in d["dram__bytes_read.sum"] else 1)
                wr = float(d["dram__bytes_write.sum"].split()[0]) * (1e6 if "Mbyte" in d["dram__bytes_write.sum"] else 1)
                summary[cfg] = {"k_cast": {"dram_bytes_per_launch": rd + wr, "source": os.path.basename(rep)}}
        launches = os.path.join(OUT, f"{TAG}_launches_{cfg}.csv")
        if os.path.exists(launches):
            import shutil
            shutil.copy(launches, os.path.join(PROF, os.path.basename(launches)))
            txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), launches],
                                 capture_output=True, text=True).stdout
            with open(os.path.join(PROF, f"{TAG}_launches_{cfg}.txt"), "w") as f:
                f.write(f"# one full step ({cfg}): per-launch device time (ncu, cold cache, serialised)\n" + txt)
    for name in ("build_C2", "build_C3", "vox_G2"):
        rep = os.path.join(OUT, f"{TAG}_{name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        for d in raw(rep):
            lines.append(f"## {name} {d['kernel']}")
            lines += [f"  {k:70s} {v}" for k, v in d.items() if k not in ("kernel", "top_stalls")]
            lines.append(f"  top stalls: {d['top_stalls']}")
            if name == "vox_G2" and "k_voxelize" in d["kernel"]:
                rd = float(d["dram__bytes_read.sum"].split()[0]) * (1e6 if "Mbyte" in d["dram__bytes_read.sum"] else 1)
                wr = float(d["dram__bytes_write.sum"].split()[0]) * (1e6 if "Mbyte" in d["dram__bytes_write.sum"] else 1)
                summary["G2"] = {"k_voxelize": {"dram_bytes_per_launch": rd + wr, "source": os.path.basename(rep)}}
    with open(os.path.join(PROF, f"{TAG}_ncu_full.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    old = {}
    p = os.path.join(PROF, "ncu_summary.json")
    if os.path.exists(p):
        old = json.load(open(p))
    old.update(summary)
    json.dump(old, open(p, "w"), indent=1)
    cj = os.path.join(OUT, f"{TAG}_configs.jsonl")
    if os.path.exists(cj):
        import shutil
        shutil.copy(cj, os.path.join(PROF, f"{TAG}_configs.jsonl"))
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
