"""Per-kernel registers / spills from a verbose build (dev tool).

    python -m paper_1805_12498_b200.build -v 2>&1 | python tools/ptxas_regs.py [regex]
"""
import re
import subprocess
import sys

pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
cur = None
spill = ""
for ln in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        spill = f"spill {m.group(1)}/{m.group(2)}"
        continue
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur and pat.search(cur):
        print(f"{m.group(1):>4} regs  {spill:>16}  {cur[:90]}")
        cur = None
