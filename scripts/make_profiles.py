"""Turn a round's gpurun_out/ evidence into the committed profiles/ summaries:
  python scripts/make_profiles.py r02
launch lists -> r02_launches_*_summary.txt (per kernel class, per level),
ncu_traffic.json / ncu_traffic_det.json (bench.py's `traffic`), full ncu
captures -> r02_ncu_*.txt (key metrics + hottest source lines), the pytest
log and the bench lines."""
import shutil, subprocess, sys
from pathlib import Path

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = Path("gpurun_out"), Path("profiles")
py = sys.executable


def run(*args):
    return subprocess.run([py, *args], capture_output=True, text=True).stdout


for mode in ("fast", "det", "rmat22"):
    csv = G / f"{tag}_launches_{mode}.csv"
    if not csv.exists():
        continue
    tj = {"fast": "ncu_traffic.json", "det": "ncu_traffic_det.json"}.get(mode, f"{tag}_ncu_traffic_{mode}.json")
    out = run("scripts/ncu_traffic.py", str(csv), str(P / tj))
    out += "\n" + run("scripts/ncu_levels.py", str(csv))
    (P / f"{tag}_launches_{mode}_summary.txt").write_text(out)
    print("wrote", P / f"{tag}_launches_{mode}_summary.txt")
for rep in sorted(G.glob(f"{tag}_k_level_*.ncu-rep")):
    out = run("scripts/ncu_summary.py", str(rep)) + "\n" + run("scripts/ncu_hotlines.py", str(rep), "30")
    (P / (rep.stem.replace("k_level", "ncu_k_level") + ".txt")).write_text(out)
    print("wrote", rep.stem)
for src, dst in (("pytest_gpu.log", f"{tag}_pytest_gpu.log"), ("bench.log", f"{tag}_bench.json"),
                 ("bench_ref.log", f"{tag}_bench_reference.json"), ("smoke.log", f"{tag}_smoke.log")):
    if (G / src).exists():
        shutil.copy(G / src, P / dst)
        print("copied", dst)
