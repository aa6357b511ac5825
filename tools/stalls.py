"""Profiling tool: aggregate ncu cuda,sass source-page stall samples per source line."""
import csv, sys, collections
rows = csv.reader(open(sys.argv[1]))
cur = None; hdr = None; agg = collections.Counter(); inst = collections.Counter(); src = {}
filet = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': continue
    if r[0] == 'Line No': hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr is None or r[0] == '': continue
    try:
        s = int(r[4]); n = int(r[7])
    except ValueError:
        continue
    agg[(cur, int(r[0]))] += s; inst[(cur, int(r[0]))] += n; src[(cur, int(r[0]))] = r[1][:90]
    filet[cur] += s
tot = sum(agg.values())
print('total samples', tot)
for f, v in filet.most_common(): print('  %-16s %5.1f%%' % (f, 100 * v / tot))
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 50):
    print('%5.2f%% %9d %-14s %5d  %s' % (100 * v / tot, inst[k], k[0], k[1], src[k]))
