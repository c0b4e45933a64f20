"""The reference's own test suite (pkg/tests: 158 unit tests + 11 acceptance
criteria) run against the GPU path through the drop-in binding
(paper_2304_13194_b200/compat/jetpart: the reference package with every
hot-path entry point rebound to this package, deterministic mode).

The suite lives in baseline/_ref/jetpart_tests next to the reference install
(git-ignored; `__graft_entry__.build()` installs both when /root/reference is
present). The run happens in a subprocess so the `jetpart` name is bound only
there. Tests that inspect the reference's CPU-only internals are listed in
EXPECTED_DIFF with the reason; everything else must pass."""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "baseline" / "_ref" / "jetpart_tests"
COMPAT = ROOT / "paper_2304_13194_b200" / "compat"

# test id -> why it cannot hold on the GPU path
EXPECTED_DIFF = {
    # The ConnectivityTable's open-addressing layout (conn.py:85-194: slot
    # regions, capacity growth on overflow, the keys array) is not modelled:
    # the GPU rebuilds conn rows on chip in every pass and only their nonzero
    # contents are observable by the partition. Every
    # content test of test_conn.py passes.
    "test_conn.py::TestRebuild::test_overflow_grows_capacity":
        "row capacity is the fixed Eq. 9 bound min(deg, k), not a growing hash table",
    "test_conn.py::TestRebuild::test_stale_zero_entries_purged_on_rebuild":
        "reads the hash table's keys/region arrays",
    # The test starts `python -m jetpart.cli` with an environment holding only
    # PATH and the thread counts, so no binding on PYTHONPATH is visible there
    # (it would run nothing of ours); test_cli_deterministic_across_threads
    # below repeats it with the binding on the path.
    "test_acceptance.py::test_11_deterministic_across_thread_counts":
        "subprocess environment drops PYTHONPATH",
}


def run_suite(*args, timeout=3000):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(COMPAT), str(ROOT), str(SUITE)])
    env["JETPART_REFERENCE"] = str(ROOT / "baseline" / "_ref")
    cmd = [sys.executable, "-m", "pytest", str(SUITE), "-q", "-rfE", "-p", "no:cacheprovider",
           "--rootdir", str(SUITE), *args]
    return subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout,
                          cwd=str(SUITE))


@pytest.mark.gpu
def test_reference_suite_on_gpu_path():
    if not SUITE.exists():
        pytest.skip("reference suite not installed (baseline/_ref/jetpart_tests)")
    p = run_suite()
    out = p.stdout + p.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "reference_suite.log").write_text(out)
    failed = set(re.findall(r"^(?:FAILED|ERROR) (\S+)", out, re.M))
    unexpected = sorted(f for f in failed if f.split(" ")[0] not in EXPECTED_DIFF)
    assert not unexpected, "\n".join(unexpected) + "\n" + out[-3000:]
    assert re.search(r"(\d+) passed", out), out[-2000:]


@pytest.mark.gpu
def test_cli_deterministic_across_threads(tmp_path):
    """Acceptance 11 (test_acceptance.py:334-354) with the binding visible:
    the reference CLI on the GPU path gives byte-identical partition files
    across thread counts and repeats."""
    if not SUITE.exists():
        pytest.skip("reference not installed")
    env0 = {"PATH": os.environ.get("PATH", "/usr/bin:/bin"),
            "PYTHONPATH": os.pathsep.join([str(COMPAT), str(ROOT)]),
            "JETPART_REFERENCE": str(ROOT / "baseline" / "_ref")}
    code = ("import sys; sys.path[:0] = [%r, %r]; import jetpart; "
            "from jetpart.generators import grid_graph; from jetpart.io import write_metis; "
            "write_metis(grid_graph(48, 48), sys.argv[1])") % (str(COMPAT), str(ROOT))
    gfile = tmp_path / "det.graph"
    subprocess.run([sys.executable, "-c", code, str(gfile)], env=env0, check=True, timeout=300)
    blobs = []
    for threads in ("1", "8"):
        for rep in ("a", "b"):
            out = tmp_path / f"p_{threads}_{rep}.txt"
            env = dict(env0, OMP_NUM_THREADS=threads, OPENBLAS_NUM_THREADS=threads)
            p = subprocess.run([sys.executable, "-m", "jetpart.cli", str(gfile), "--k", "8",
                                "--seed", "7", "--deterministic", "--out", str(out)],
                               env=env, capture_output=True, text=True, timeout=300)
            assert p.returncode == 0, p.stderr
            blobs.append(out.read_bytes())
    assert all(b == blobs[0] for b in blobs)
