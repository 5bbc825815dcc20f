"""Per-kernel metric table from an ncu --csv launch log (dev tool).

    python tools/ncu_csv.py log.csv [name-regex]
"""
import collections
import csv
import re
import sys

pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tab = collections.OrderedDict()
for r in rows:
    if len(r) > 10 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if not pat.search(d["Kernel Name"]):
            continue
        key = (d["ID"], d["Kernel Name"].split("(")[0])
        tab.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"].replace(",", "")
tot = 0.0
for (i, k), m in tab.items():
    t = float(m.get("gpu__time_duration.sum", 0)) / 1e6
    tot += t
    extra = "  ".join(f"{n.split('.')[0].split('__')[-1]}={v}" for n, v in m.items() if n != "gpu__time_duration.sum")
    print(f"{k[:46]:46s} {t:10.3f} ms  {extra}")
print(f"total {tot:.1f} ms")
