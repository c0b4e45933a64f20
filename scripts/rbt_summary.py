import re, collections, sys
d = collections.defaultdict(list)
for l in open(sys.argv[1]):
    m = re.match(r'RBT s=(\d) L=(\d+) path=(\d) sort=(\d+) mid=(\d+) out=(\d+)', l)
    if not m:
        continue
    s, L, p, a, b, c = map(int, m.groups())
    d[(s, p, min(13, L.bit_length()))].append((a, b, c))
for k in sorted(d):
    v = d[k]
    n = len(v)
    print("strong=%d path=%d log2L=%d n=%d" % (k + (n,)), [round(sum(x[i] for x in v) / n) for i in range(3)])
