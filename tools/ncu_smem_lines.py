"""Attribute shared-memory wavefronts (L1 Wavefronts Shared) to CUDA source lines (dev tool).

usage: ncu_lines.py <report.ncu-rep> <object.o> <mangled-kernel-name> [topN]
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-fun", fn, cubin], capture_output=True, text=True).stdout
if not dis:
    dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
# offset -> source line (innermost)
line_of = {}
cur = None
in_fn = False
for ln in dis.splitlines():
    if re.match(r"\s*\.text\." + re.escape(fn) + r":", ln) or (".text." + fn + ":") in ln:
        in_fn = True
        continue
    if in_fn and re.match(r"\s*\.text\.", ln) and fn not in ln:
        in_fn = False
    m = re.search(r'## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*)", ln)
    if m and in_fn:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) > 5]
base = int(data[0][ix["Address"]], 16)
samp = collections.Counter()
inst = collections.Counter()
tot = 0
for r in data:
    off = int(r[ix["Address"]], 16) - base
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    key = line_of.get(off, "?")
    samp[key] += int(r[ix["L1 Wavefronts Shared"]] or 0)
    inst[key] += n
    tot += int(r[ix["L1 Wavefronts Shared"]] or 0)
src = {}
for k, v in samp.most_common(top):
    print(f"{100 * v / tot:5.1f}%  inst={inst[k]:11d}  {k}")
