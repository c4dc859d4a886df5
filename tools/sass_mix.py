"""Summarise an ncu --page source --print-source sass CSV: instruction mix,
stall samples and shared-memory wavefronts per SASS opcode."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS = h.index('Source'); iE = h.index('Instructions Executed'); iW = h.index('Warp Stall Sampling (All Samples)')
iC = h.index('L1 Wavefronts Shared'); iI = h.index('L1 Wavefronts Shared Ideal')
op = collections.Counter(); st = collections.Counter(); wf = collections.Counter(); wfi = collections.Counter()
tot = stot = 0
for r in rows[2:]:
    if len(r) <= iI or r[iE] == 'Instructions Executed':
        continue
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_.]+)', r[iS].strip())
    if not m:
        continue
    o = m.group(2).split('.')[0]
    try:
        e = int(float(r[iE] or 0)); s = int(float(r[iW] or 0))
    except ValueError:
        continue
    op[o] += e; st[o] += s; tot += e; stot += s
    wf[o] += int(float(r[iC] or 0)); wfi[o] += int(float(r[iI] or 0))
for o, c in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {c / tot * 100:6.2f}% inst  {st[o] / max(stot, 1) * 100:6.2f}% stall  wf={wf[o]} ideal={wfi[o]}")
print("total warp-instructions", tot)
