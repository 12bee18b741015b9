"""Summarise an ncu launch list CSV (gpu__time_duration.sum per launch): one build + cast sequence."""
import csv, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith('==')))
h = rows[0]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
seq = [(r[ki].split('(')[0].replace('fgl::<unnamed>::', '').replace('void ', '')[:48], float(r[vi].replace(',', '')) / 1e3)
       for r in rows[1:] if len(r) > vi]
starts = [i for i, (k, _) in enumerate(seq) if k.startswith('k_validate')]
i0 = starts[min(1, len(starts) - 1)]
end = next((i for i in range(i0 + 1, len(seq)) if seq[i][0].startswith('k_validate')), len(seq))
tot = 0
for k, v in seq[i0:end]:
    print(f"  {k:48s} {v:9.1f} us")
    tot += v
print(f"  {'total':48s} {tot:9.1f} us")
