"""Round-2 summaries of the gpurun_out/ artefacts of tools/r02_profile.sh into profiles/:
per-config cast-kernel ncu tables, ncu_summary.json (the fields bench.py's roofline reads), launch
lists, the C3 build kernels, the sanitizer log and the bench lines."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
# rays per launch of the profiled cast (tools/r02_profile.sh workloads)
RAYS = {"C2": 64 * 64 * 2048, "C3": 128 * 2048, "C4": 20 * 20000, "C5": 256 * 64 * 2048}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_local_op_st.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                d[k] = (r[h.index(k)], units[h.index(k)])
        st = [(float(r[i]), x) for i, x in enumerate(h) if x.startswith("smsp__average_warps_issue_stalled")
              and x.endswith("_per_issue_active.ratio") and r[i] not in ("", "0")]
        d["top_stalls"] = {x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: v
                           for v, x in sorted(st, reverse=True)[:6]}
        res.append(d)
    return res


def val(d, k):
    v, u = d[k]
    x = float(v.replace(",", ""))
    return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9,
                "msecond": 1e-3, "ms": 1e-3}.get(u, 1.0)


def main():
    summary = {}
    lines = [f"# {TAG}: ncu --set full of one k_cast_dyn launch per config (tools/r02_profile.sh)"]
    for cfg, rays in RAYS.items():
        rep = os.path.join(OUT, f"{TAG}_k_cast_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        for d in raw(rep):
            inst = val(d, "smsp__inst_executed.sum")
            simt = val(d, "smsp__thread_inst_executed_per_inst_executed.ratio")
            lines.append(f"## {cfg} {d['kernel']}  ({rays} rays per launch)")
            lines += [f"  {k:72s} {v[0]} {v[1]}" for k, v in d.items() if k not in ("kernel", "top_stalls")]
            lines.append(f"  thread instructions per ray {inst * simt / rays:.0f}; lane slots per ray "
                         f"{inst * 32 / rays:.0f}")
            lines.append(f"  top stalls (warps per issued instruction): {d['top_stalls']}")
            summary.setdefault(cfg, {})["k_cast"] = {
                "dram_bytes_per_launch": val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum"),
                "issue_slot_frac": val(d, "sm__inst_issued.avg.pct_of_peak_sustained_active") / 100,
                "thread_inst_per_ray": inst * simt / rays, "lane_slots_per_ray": inst * 32 / rays,
                "simt_lanes": simt,
                "l1_data_pipe_frac": val(d, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed") / 100,
                "duration_us": val(d, "gpu__time_duration.sum") * 1e6, "source": os.path.basename(rep)}
        launches = os.path.join(OUT, f"{TAG}_launches_{cfg}.csv")
        if os.path.exists(launches):
            shutil.copy(launches, os.path.join(PROF, os.path.basename(launches)))
            txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), launches],
                                 capture_output=True, text=True).stdout
            with open(os.path.join(PROF, f"{TAG}_launches_{cfg}.txt"), "w") as f:
                f.write(f"# one full step ({cfg}): per-launch device time (ncu, cold cache, serialised)\n" + txt)
    with open(os.path.join(PROF, f"{TAG}_ncu_cast.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    # keep earlier configs (e.g. G2) already in the summary
    path = os.path.join(PROF, "ncu_summary.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    for cfg, v in summary.items():
        old.setdefault(cfg, {}).update(v)
    with open(path, "w") as f:
        json.dump(old, f, indent=1)
    rep = os.path.join(OUT, f"{TAG}_build_C3.ncu-rep")
    if os.path.exists(rep):
        bl = [f"# {TAG}: every kernel of one warm C3 (10 M triangles) build, ncu --set full"]
        bl.append(f"{'kernel':34s} {'us':>8s} {'issue%':>7s} {'warps%':>7s} {'dramR MB':>9s} {'dramW MB':>9s} "
                  f"{'winst M':>8s} {'L1hit':>6s} {'L2hit':>6s} {'regs':>5s}")
        for d in raw(rep):
            bl.append(f"{d['kernel'][:34]:34s} {val(d, 'gpu__time_duration.sum') * 1e6:8.1f} "
                      f"{val(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):7.1f} "
                      f"{val(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):7.1f} "
                      f"{val(d, 'dram__bytes_read.sum') / 1e6:9.1f} {val(d, 'dram__bytes_write.sum') / 1e6:9.1f} "
                      f"{val(d, 'smsp__inst_executed.sum') / 1e6:8.1f} {val(d, 'l1tex__t_sector_hit_rate.pct'):6.1f} "
                      f"{val(d, 'lts__t_sector_hit_rate.pct'):6.1f} {val(d, 'launch__registers_per_thread'):5.0f}")
        with open(os.path.join(PROF, f"{TAG}_ncu_build_C3.txt"), "w") as f:
            f.write("\n".join(bl) + "\n")
    for name in (f"{TAG}_sanitizer.txt", f"{TAG}_configs.jsonl"):
        p = os.path.join(OUT, name)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(PROF, name))
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
