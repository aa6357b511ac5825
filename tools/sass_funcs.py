"""Profiling tool: static SASS instructions of one kernel attributed to the
engine source function of each instruction's line (nvdisasm -g of the
shipped library).   python tools/sass_funcs.py <all.sass from nvdisasm -g -c> <kernel substring> [N]"""
import collections
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import ncu_regions as R  # noqa: E402

funcs = {}


def owner(path, line):
    if path not in funcs:
        p = Path(path)
        funcs[path] = R.functions_of(p) if p.exists() else []
    return R.owner(funcs[path], line)


sec = cur = None
cnt = collections.Counter()
for ln in open(sys.argv[1]):
    if ln.startswith('.text.'):
        sec = ln.strip()[6:-1]
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    if sec and sys.argv[2] in sec and re.match(r'\s+/\*[0-9a-f]{4,}\*/', ln) and cur:
        cnt[(Path(cur[0]).name, owner(cur[0], cur[1]))] += 1
tot = sum(cnt.values())
print('total', tot)
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print('%6d %5.1f%% %s' % (v, 100 * v / tot, k))
