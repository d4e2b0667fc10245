"""Instruction mix and stall samples by SASS opcode from an ncu --page source --csv export."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter(); st = collections.Counter()
tot_ex = tot_st = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    try:
        e = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    ex[o] += n; st[o] += e; tot_ex += n; tot_st += e
print(f"total warp instructions {tot_ex}, stall samples {tot_st}")
for o, n in ex.most_common(28):
    print(f"{o:12s} {n:12d} {n / tot_ex:6.1%}   stall samples {st[o] / max(tot_st, 1):6.1%}")
