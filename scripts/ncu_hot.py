"""Group an ncu --page source --csv --print-source sass export into runs of
instructions with equal execution counts (basic blocks), print the heavy ones.

    python scripts/ncu_hot.py src.csv [min_share]
"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1]))]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ia, isrc = hdr.index('Address'), hdr.index('Source')
ie, iss = hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
iwf = hdr.index('L1 Wavefronts Shared') if 'L1 Wavefronts Shared' in hdr else None
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[ie]) for r in data)
stot = sum(num(r[iss]) for r in data)
print('total warp inst', tot, 'samples', stot)
blocks, cur = [], None
for r in data:
    c = num(r[ie])
    if cur is None or c != cur['c']:
        cur = {'a': r[ia][-5:], 's': r[isrc].strip()[:44], 'c': c, 'n': 0, 'acc': 0, 'samp': 0, 'wf': 0}
        blocks.append(cur)
    cur['n'] += 1
    cur['acc'] += c
    cur['samp'] += num(r[iss])
    if iwf is not None:
        cur['wf'] += num(r[iwf])
for b in blocks:
    if b['acc'] > tot * thr or b['samp'] > stot * thr:
        print(f"{b['a']} {b['s']:44s} n={b['n']:4d} each={b['c']:>10d} inst={100*b['acc']/tot:5.1f}% "
              f"stall={100*b['samp']/max(stot,1):5.1f}% smem_wf={b['wf']}")
