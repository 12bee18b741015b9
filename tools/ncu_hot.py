"""Hottest SASS lines (warp-stall samples) of one kernel in an .ncu-rep:
python tools/ncu_hot.py rep.ncu-rep kernel_regex [n]"""
import csv, io, subprocess, sys

out = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass",
                               "-k", "regex:" + sys.argv[2]], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Address" in r][0]
h = rows[hi]
data, seen = [], set()
for r in rows[hi + 1:]:
    if len(r) != len(h):
        if data:
            break  # next kernel
        continue
    d = dict(zip(h, r))
    if d["Address"] in seen:
        continue
    seen.add(d["Address"])
    try:
        s, ie = int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"])
    except ValueError:
        continue
    data.append((s, ie, d["Address"][-5:], d["Source"][:72]))
tot = sum(x[0] for x in data)
print("samples", tot, "warp inst", sum(x[1] for x in data))
for x in sorted(data, reverse=True)[: int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{x[0]:7d} {100 * x[0] / max(tot, 1):5.1f}% {x[1]:10d}  {x[2]}  {x[3]}")
