"""Summarise an ncu launch-list CSV: per kernel, and per refinement level
(the sequence is split at every k_project launch)."""
import collections, csv, io, re, sys
path = sys.argv[1]
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
L = collections.OrderedDict()
for r in rows:
    d = L.setdefault(r['ID'], {'name': r['Kernel Name'], 'grid': r['Grid Size']})
    v = r['Metric Value'].replace(',', '')
    d[r['Metric Name']] = float(v) if v else 0.0
def short(n):
    m = re.match(r'(?:void )?(?:jet::)?(\w+)(<[^(]*)?', n)
    s = m.group(1) if m else n[:40]
    if m and m.group(2):
        t = m.group(2)
        t = t.replace('jet::', '')
        s += t[:24]
    return s
seq = list(L.values())
levels, cur = [], []
for d in seq:
    if short(d['name']).startswith('k_project'):
        levels.append(cur); cur = []
    cur.append(d)
levels.append(cur)
tot = sum(d['gpu__time_duration.sum'] for d in seq)
print(f"launches {len(seq)} total {tot/1e6:.2f} ms")
names = ["coarsen+init+top"] + [f"L{len(levels)-1-i-1}" for i in range(len(levels)-1)]
for nm, lv in zip(names, levels):
    t = sum(d['gpu__time_duration.sum'] for d in lv)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in lv:
        a = agg[short(d['name'])]; a[0] += 1; a[1] += d['gpu__time_duration.sum']
        a[2] += d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    top = sorted(agg.items(), key=lambda x: -x[1][1])[:6]
    print(f"{nm:18s} {len(lv):5d} launches {t/1e6:8.2f} ms | " +
          "  ".join(f"{k}:{v[0]}x{v[1]/v[0]/1e3:.0f}us" for k, v in top))
