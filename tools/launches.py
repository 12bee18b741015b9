"""Summarise an ncu launch list CSV (gpu__time_duration.sum per launch): one build + cast sequence."""
import csv, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith('==')))
h = rows[0]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
seq = [(r[ki].split('(')[0].replace('fgl::<unnamed>::', '').replace('void ', '')[:48], float(r[vi].replace(',', '')) / 1e3)
       for r in rows[1:] if len(r) > vi and 'at::' not in r[ki]]  # torch kernels = the untimed L2 flush
# a step starts at the upload's validation kernel (k_validate; a Gaussian scene runs k_gauss_prep
# twice per step: upload validation + build)
mark, per = ('k_validate', 1) if any(k.startswith('k_validate') for k, _ in seq) else ('k_gauss_prep', 2)
starts = [i for i, (k, _) in enumerate(seq) if k.startswith(mark)]
i0 = starts[min(per, len(starts) - 1)]
end = starts[2 * per] if len(starts) > 2 * per else len(seq)
tot = 0
for k, v in seq[i0:end]:
    print(f"  {k:48s} {v:9.1f} us")
    tot += v
print(f"  {'total':48s} {tot:9.1f} us")
