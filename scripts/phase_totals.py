"""Sum the JET_PHASES per-phase times (us/pass x passes) of the last repetition in a probe log."""
import re, collections, sys
tot = collections.Counter()
lines = [l for l in open(sys.argv[1]) if l.startswith('PHASES')]
idx = max(i for i, l in enumerate(lines) if l.startswith('PHASES L17') or l.startswith('PHASES L14'))
first = lines[idx].split()[1]
start = idx
while start > 0 and lines[start - 1].split()[1] == first:
    start -= 1
for l in lines[start:]:
    m = re.match(r'PHASES L(\d+) blocks=\d+ (\w+) x(\d+) \(us/pass\): (.*)', l)
    L, kind, cnt, rest = m.groups()
    for k, v in re.findall(r'(\w[\w+]*)=([\d.]+)', rest):
        tot[(kind, k)] += float(v) * int(cnt)
for k, v in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 16):
    print("%-8s %-14s %7.2f ms" % (k[0], k[1], v / 1000))
print("total %.2f ms" % (sum(tot.values()) / 1000))
