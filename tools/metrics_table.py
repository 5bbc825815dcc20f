"""Summarise tools/ncu_metrics.sh output: one row per kernel launch."""
import csv
import re
import sys
from collections import OrderedDict
from math import comb

sys.path.insert(0, '.')
from paper_1805_12498_b200 import costmodel as c  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]
ix = {k: hdr.index(k) for k in ('ID', 'Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit')}
launches = OrderedDict()
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    d = launches.setdefault(r[ix['ID']], {'name': r[ix['Kernel Name']]})
    v = r[ix['Metric Value']].replace(',', '')
    try:
        v = float(v)
    except ValueError:
        pass
    d[r[ix['Metric Name']]] = (v, r[ix['Metric Unit']])
D = 26
print(f"{'kernel':28s} {'ms':>8s} {'fp64pipe%':>9s} {'issue%':>7s} {'occ%':>6s} {'regs':>5s} "
      f"{'instr/DFMA':>10s} {'bankconf/wavefr':>15s} {'exec TF/s':>9s} {'alg TF/s':>8s}")
for d in launches.values():
    m = re.search(r'(\w+_term_kernel)<(\d+)', d['name'])
    if not m:
        continue
    S = int(m.group(2))
    t, unit = d['gpu__time_duration.sum']
    t *= {'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3, 'second': 1.0}.get(unit, 1e-9)
    g = lambda k: d.get(k, (0.0, ''))[0]  # noqa: E731
    dfma = g('sm__sass_thread_inst_executed_op_dfma_pred_on.sum')
    dadd = g('sm__sass_thread_inst_executed_op_dadd_pred_on.sum')
    dmul = g('sm__sass_thread_inst_executed_op_dmul_pred_on.sum')
    execf = 2 * dfma + dadd + dmul
    algf = comb(D, S // 2) * c.cma(S, D) * 8
    conf = g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum') + g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum')
    wav = g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')
    ipd = g('sm__inst_executed.sum') / max(1.0, g('sm__inst_executed_pipe_fp64.sum'))
    print(f"{m.group(1)[:20] + '<' + str(S) + '>':28s} {t*1e3:8.2f} "
          f"{g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):9.1f} "
          f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):7.1f} "
          f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} {g('launch__registers_per_thread'):5.0f} "
          f"{ipd:10.2f} {conf / max(1.0, wav):15.3f} {execf / t / 1e12:9.2f} {algf / t / 1e12:8.2f}")
