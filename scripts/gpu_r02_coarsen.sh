mkdir -p gpurun_out
JET_MODE=fast JET_MATCH_STATS=1 JET_COARSEN_TIMES=1 JET_SYNC_STATS=1 timeout 300 python scripts/one_partition.py 128 64 2 > gpurun_out/coarsen128.log 2>&1
grep -E "COARSEN|SYNC" gpurun_out/coarsen128.log | tail -22
python - <<'PY'
import re, collections
rounds = collections.OrderedDict()
lines = open('gpurun_out/coarsen128.log').read().splitlines()
half = len([l for l in lines if l.startswith('FAST')]) // 2
cnt = 0
for l in lines:
    m = re.match(r'FAST n=(\d+) round=(\d+) proposers=(\d+) pairs=(\d+)', l)
    if m:
        cnt += 1
        if cnt <= half: continue
        n, r, p, q = map(int, m.groups()); rounds.setdefault(n, []).append((p, q))
for n, v in rounds.items(): print(n, len(v), v)
PY
