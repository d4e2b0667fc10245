"""Aggregate an ncu --page source --csv (SASS view) by opcode: executed warp instructions and stall samples."""
import csv, sys, re
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; idx = {k: i for i, k in enumerate(h)}
def f(x):
    try: return float(x)
    except: return 0.0
agg = defaultdict(lambda: [0.0, 0.0])
tot = [0.0, 0.0]
lines = []
for r in rows[2:]:
    if len(r) < len(h): continue
    src = r[idx['Source']].strip()
    op = re.sub(r'^@!?U?P\w+\s+', '', src).split(' ')[0].split('.')[0]
    ie, st = f(r[idx['Instructions Executed']]), f(r[idx['Warp Stall Sampling (All Samples)']])
    agg[op][0] += ie; agg[op][1] += st; tot[0] += ie; tot[1] += st
    lines.append((ie, st, r[idx['Address']], src))
print('total warp insts %.0f, stall samples %.0f' % tuple(tot))
for op, (ie, st) in sorted(agg.items(), key=lambda t: -t[1][0])[:25]:
    print('%-10s %6.2f%% inst  %6.2f%% stall' % (op, 100 * ie / tot[0], 100 * st / max(tot[1], 1)))
if len(sys.argv) > 2:
    print('--- top stall lines')
    for ie, st, a, s in sorted(lines, key=lambda t: -t[1])[:int(sys.argv[2])]:
        print('%8.0f %6.0f %s %s' % (ie, st, a[-5:], s[:90]))
