"""Summarise an ncu source-page CSV (SASS) by barrier-delimited regions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
iS = hdr.index('Warp Stall Sampling (All Samples)')
iE = hdr.index('Instructions Executed')
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(int(r[iS] or 0) for r in data)
print("total samples", tot, "total inst %.3fe9" % (sum(int(r[iE] or 0) for r in data) / 1e9), "code lines", len(data))
reg = []
cur = {'start': 0, 'samples': 0, 'inst': 0, 'n': 0, 'stalls': {}}
for k, r in enumerate(data):
    cur['samples'] += int(r[iS] or 0)
    cur['inst'] += int(r[iE] or 0)
    cur['n'] += 1
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            cur['stalls'][hdr[i]] = cur['stalls'].get(hdr[i], 0) + v
    if 'BAR.SYNC' in r[1] or 'EXIT' in r[1]:
        cur['end'] = k
        reg.append(cur)
        cur = {'start': k + 1, 'samples': 0, 'inst': 0, 'n': 0, 'stalls': {}}
reg.append(cur)
for g in reg:
    if g['samples'] > tot * 0.005:
        top = sorted(g['stalls'].items(), key=lambda x: -x[1])[:6]
        print(f"lines {g['start']}-{g.get('end')}: {g['n']} instrs, samples {100 * g['samples'] / tot:.1f}%, "
              f"executed {g['inst'] / 1e9:.2f}e9", [(a[6:], round(100 * b / tot, 1)) for a, b in top])

# hottest instructions
top = sorted(range(len(data)), key=lambda k: -int(data[k][iS] or 0))[:15]
for k in top:
    st = sorted(((hdr[i][6:], int(data[k][i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:2]
    print(f"  line {k}: {data[k][1].strip()[:50]:50s} {100 * int(data[k][iS]) / tot:5.1f}%  exec {data[k][iE]}  {st}")
