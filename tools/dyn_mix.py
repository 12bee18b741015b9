"""Dynamic instruction mix of k_cast_dyn from an ncu --set full --import-source capture: executed
warp instructions per opcode class and per code region (ray setup, descent, leaf phase, write),
memory instructions that matter (256-bit node loads, triangle loads, local-memory stack), lanes
active per region. Usage: tools/dyn_mix.py report.ncu-rep rays_per_launch"""
import collections
import csv
import re
import subprocess
import sys

rep, rays = sys.argv[1], int(sys.argv[2])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:k_cast_dyn"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
R = [r for r in rows[hi + 1:] if len(r) == len(h)]
ia, it = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
tot = sum(int(r[ia]) for r in R)
CLASSES = [("FP32 FFMA/FMUL/FADD", r"^(FFMA|FMUL|FADD)"), ("FP32 FMNMX/FMNMX3", r"^FMNMX"), ("FSETP/FSEL", r"^(FSETP|FSEL)"),
           ("MUFU", r"^MUFU"), ("integer / move", r"^(IADD|IMAD|ISETP|LOP|SHF|SEL|PRMT|VIADD|VIMNMX|LEA|POPC|FLO|BREV|MOV|CS2R|S2R|LDC|UMOV|U)"),
           ("control (BRA/BSSY/BSYNC/VOTE/...)", r"^(BRA|BSSY|BSYNC|WARPSYNC|VOTE|BREAK|EXIT|RET|CALL|YIELD|BRX|NOP|PLOP|SHFL)"),
           ("LDG (global loads)", r"^LDG"), ("STG", r"^STG"), ("LDL/STL (stack)", r"^(LDL|STL)"), ("ATOM", r"^(ATOM|RED)")]
cls = collections.Counter()
mem = collections.Counter()
for r in R:
    t = r[1].strip()
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    n = int(r[ia])
    for c, rx in CLASSES:
        if re.match(rx, op):
            cls[c] += n
            break
    else:
        cls["other"] += n
    if op.startswith(("LDG", "LDL", "STL", "STG")):
        mem[op] += n
print(f"# dynamic instruction mix of k_cast_dyn ({rep}); {tot / 1e6:.1f} M warp instructions per launch, "
      f"{tot * 32 / rays:.0f} lane slots per ray ({rays} rays)")
print(f"{'class':36s} {'warp instr / ray-tile':>22s} {'share':>7s}")
for c, _ in CLASSES + [("other", "")]:
    if cls[c]:
        print(f"{c:36s} {cls[c] * 32 / rays:22.1f} {cls[c] / tot * 100:6.1f}%")
print("\nmemory instructions (executed warp instructions per 32-ray tile)")
for op, n in sorted(mem.items(), key=lambda x: -x[1]):
    print(f"  {op:34s} {n * 32 / rays:8.2f}")
