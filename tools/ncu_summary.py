"""Print the key ncu 'details' metrics of a report (dev tool)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
for r in rows[1:]:
    if len(r) < 15 or not r[ix["Metric Name"]]:
        continue
    print(f'{r[ix["Section Name"]][:26]:26s} | {r[ix["Metric Name"]][:46]:46s} | {r[ix["Metric Value"]]:>14s} {r[ix["Metric Unit"]]}')
