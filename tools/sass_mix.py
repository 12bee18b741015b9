"""Static SASS instruction mix of the cast kernels in libfgl.so (cuobjdump; no GPU needed):
per kernel the instruction count by class and the memory instructions that matter for the traversal
(256-bit node loads, 128-bit triangle loads, local-memory stack traffic). Writes a text table."""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2509_17390_b200/libfgl.so"
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
WANT = ("k_cast_dynINS0_7SpinGenELb0ELi2", "k_cast_dynINS0_7SpinGenELb0ELi8", "k_cast_dynINS0_10RosetteGenELb0ELi2")
CLASSES = [("FFMA/FMUL/FADD", r"^(FFMA|FMUL|FADD)"), ("FMNMX/FMNMX3", r"^FMNMX"), ("FSETP/FSEL", r"^(FSETP|FSEL)"),
           ("integer ALU", r"^(IADD|IMAD|ISETP|LOP|SHF|SEL|PRMT|VIADD|VIMNMX|LEA|IABS|POPC|FLO|BREV)"),
           ("MUFU", r"^MUFU"), ("branch/sync", r"^(BRA|BSSY|BSYNC|WARPSYNC|VOTE|BREAK|EXIT|RET|CALL|YIELD|BRX|NOP)"),
           ("LDG", r"^LDG"), ("STG", r"^STG"), ("LDL/STL", r"^(LDL|STL)"), ("LDS/STS", r"^(LDS|STS)"),
           ("SHFL", r"^SHFL"), ("ATOM", r"^(ATOM|RED)")]
print(f"# static SASS mix of the cast kernels ({LIB}), tools/sass_mix.py")
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if not any(w in name for w in WANT):
        continue
    ins = []
    for ln in f.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(.*?);", ln)
        if m:
            t = m.group(1).strip()
            if t.startswith("@"):
                t = t.split(None, 1)[1]
            ins.append(t)
    ops = [i.split()[0] for i in ins]
    cls = collections.Counter()
    for o in ops:
        for cname, rx in CLASSES:
            if re.match(rx, o):
                cls[cname] += 1
                break
        else:
            cls["other"] += 1
    print(f"\n## {name}\n  total instructions: {len(ops)}")
    for cname, _ in CLASSES + [("other", "")]:
        if cls[cname]:
            print(f"  {cname:16s} {cls[cname]:5d}")
    mem = collections.Counter(o for o in ops if o.startswith(("LDG", "STG", "LDL", "STL", "LDS", "STS")))
    for o, c in sorted(mem.items()):
        print(f"    {o:34s} {c:4d}")
