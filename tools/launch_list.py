"""Print the per-launch device times of an ncu --csv launch list (gpu__time_duration.sum), even when the
program's own stdout is interleaved in the file: python tools/launch_list.py file.csv [max_rows]"""
import csv, sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 10 ** 9
for r in rows[1:lim + 1]:
    if r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("unnamed>::", "").replace("void ", "")
        print(f"  {name[:52]:52s} {float(r[vi]) / 1000:9.1f} us")
