"""Profiling tool: per-opcode executed counts and stall samples from an ncu cuda,sass source csv."""
import csv, sys, collections, re
rows = csv.reader(open(sys.argv[1]))
hdr = None; ex = collections.Counter(); st = collections.Counter(); thr = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == 'Line No': hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr is None or r[0] != '' or len(r) < 8: continue
    sass = r[3].strip()
    if not sass: continue
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?', sass)
    if not m: continue
    op = m.group(2)
    try:
        s = int(r[4]); n = int(r[7]); t = int(r[8])
    except ValueError:
        continue
    ex[op] += n; st[op] += s; thr[op] += t
tot_e = sum(ex.values()); tot_s = sum(st.values())
print('warp-instr executed %d, stall samples %d' % (tot_e, tot_s))
for op, v in ex.most_common(40):
    print('%-10s exec %8d (%4.1f%%)  thr/inst %5.2f  stall %5.1f%%' % (op, v, 100 * v / tot_e, thr[op] / max(v, 1), 100 * st[op] / tot_s))
