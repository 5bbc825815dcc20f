"""Per-class efficiency from an ncu gpu__time_duration launch list of tools/class_time.py."""
import csv
import re
import sys
from math import comb

sys.path.insert(0, '.')
from paper_1805_12498_b200 import costmodel as c  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
ki, vi, ui = rows[h].index('Kernel Name'), rows[h].index('Metric Value'), rows[h].index('Metric Unit')
D = 26
tot_t = tot_f = 0.0
for r in rows[h + 1:]:
    m = re.search(r'(fast_term_kernel|mirror_term_kernel|modp_term_kernel|terms_smem_class_kernel)<(\d+)', r[ki])
    t = float(r[vi]) * {'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3, 'second': 1.0}.get(r[ui], 1e-9)
    tot_t += t
    if not m:
        print(f"{r[ki][:40]:40s} {t*1e3:9.3f} ms")
        continue
    S = int(m.group(2))
    f = comb(D, S // 2) * c.cma(S, D) * 8
    tot_f += f
    print(f"{m.group(1)} S={S:2d} {t*1e3:9.3f} ms  {f/t/1e12:6.2f} TF/s")
print(f"total {tot_t*1e3:.1f} ms, {tot_f/tot_t/1e12:.2f} TF/s")
