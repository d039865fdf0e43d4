"""Aggregate ncu source-page stall samples (export: --page source --csv --print-source cuda,sass) by CUDA line."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur_file = None; hdr = None; agg = collections.Counter(); src = {}; cur_line = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) < 5: continue
    if r[0] and r[0].isdigit():
        cur_line = (cur_file, int(r[0])); src[cur_line] = r[1]
    s = r[4]
    if s.isdigit() and int(s) > 0 and cur_line: agg[cur_line] += int(s)
tot = sum(agg.values()); print('total samples', tot)
for k, v in agg.most_common(n): print('%5.1f%% %s:%d  %s' % (100 * v / tot, k[0], k[1], src.get(k, '').strip()[:100]))
