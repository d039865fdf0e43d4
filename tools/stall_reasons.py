"""Per-instruction stall reasons from an ncu source export (--page source --csv --print-source sass): the top
instructions by samples with their dominant reasons, and kernel-wide reason totals."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kern = int(sys.argv[3]) if len(sys.argv) > 3 else 0
blocks = []; cur = None
for r in rows:
    if r and r[0] == 'Kernel Name': cur = {'name': r[1], 'rows': []}; blocks.append(cur); continue
    if r and r[0] == 'Address': cur['hdr'] = r; continue
    if cur and r: cur['rows'].append(r)
b = blocks[kern]; h = b['hdr']
i_s = h.index('Warp Stall Sampling (All Samples)'); i_src = h.index('Source')
reasons = [i for i, x in enumerate(h) if x.startswith('stall_') and 'Not Issued' not in x]
tot = collections.Counter()
for r in b['rows']:
    for i in reasons:
        if r[i].isdigit(): tot[h[i]] += int(r[i])
T = sum(tot.values())
print(b['name'][:80]); print('reasons:', ', '.join(f'{k[6:]} {100*v/T:.1f}%' for k, v in tot.most_common(10)))
rs = sorted(b['rows'], key=lambda r: -int(r[i_s]) if r[i_s].isdigit() else 0)[:n]
for r in rs:
    rr = sorted(((int(r[i]) if r[i].isdigit() else 0, h[i][6:]) for i in reasons), reverse=True)[:3]
    print(f"{int(r[i_s]):6d} {r[0][-5:]} {r[i_src].strip()[:60]:60s} " + ' '.join(f'{k}:{v}' for v, k in rr if v))
