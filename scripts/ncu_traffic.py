"""profiles/ncu_traffic.json from an ncu launch list (--metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum): mean DRAM
bytes and duration per launch for each kernel class bench.py reports."""
import collections, csv, io, json, re, sys
CLASSES = {"k_level": "refine_level", "k_resolve": "match_resolve", "k_agg_small": "lp_sweep"}
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
L = collections.OrderedDict()
for r in rows:
    d = L.setdefault(r["ID"], {"name": r["Kernel Name"]})
    v = r["Metric Value"].replace(",", "")
    unit = r.get("Metric Unit", "")
    x = float(v) if v else 0.0
    if r["Metric Name"].startswith("dram__bytes"):
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    elif r["Metric Name"] == "gpu__time_duration.sum":
        x *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}.get(unit, 1e-9)
    d[r["Metric Name"]] = x
agg = collections.defaultdict(lambda: {"launches": 0, "bytes": 0.0, "s": 0.0})
for d in L.values():
    m = re.match(r"(?:void )?(?:jet::)?(\w+)", d["name"])
    base = m.group(1) if m else d["name"]
    cls = CLASSES.get(base, base)
    a = agg[cls]
    a["launches"] += 1
    a["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    a["s"] += d.get("gpu__time_duration.sum", 0)
out = {}
for cls, a in sorted(agg.items(), key=lambda x: -x[1]["s"]):
    out[cls] = {"launches": a["launches"], "dram_bytes_per_launch": a["bytes"] / a["launches"],
                "ms_per_launch": 1e3 * a["s"] / a["launches"],
                "dram_gbs": a["bytes"] / a["s"] / 1e9 if a["s"] else None,
                "source": sys.argv[1].split("/")[-1]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
try:
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except Exception:
    peak = 6546.6
tot_ms = sum(v["ms_per_launch"] * v["launches"] for v in out.values())
print(f"{'kernel class':24s} {'launches':>8s} {'ms/launch':>10s} {'share':>6s} {'DRAM MB/launch':>15s} {'DRAM GB/s':>10s} {'% of HBM peak':>14s}")
for k, v in list(out.items())[:16]:
    share = v["ms_per_launch"] * v["launches"] / tot_ms
    print(f"{k:24s} {v['launches']:8d} {v['ms_per_launch']:10.3f} {100*share:5.1f}% {v['dram_bytes_per_launch']/1e6:15.1f} "
          f"{v['dram_gbs'] or 0:10.1f} {100*(v['dram_gbs'] or 0)/peak:13.1f}%")
print(f"(ncu launch list: serialised, cold-cache per-launch times; peak {peak} GB/s from MEASURED_PEAKS.json)")
