"""The drop-in binding (paper_2304_13194_b200/compat/jetpart) on CPU: the
reference's modules are loaded and every hot-path name they hold is rebound
to this package (no GPU call is made here)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref" / "jetpart"

CHECK = r"""
import jetpart, jetpart.driver, jetpart.cli, jetpart.estimator, jetpart.coarsen, jetpart.conn
import jetpart.refine, jetpart.rebalance, jetpart.initpart, jetpart.graph, jetpart.errors
import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import jetpart_compat as C, ops
assert jetpart.partition is C.partition
assert jetpart.driver.partition is C.partition
assert jetpart.cli.partition is C.partition            # cli.main -> GPU
assert jetpart.estimator.partition is C.partition      # JetPartitioner.fit -> GPU
assert jetpart.coarsen.build_hierarchy is ops.build_hierarchy
assert jetpart.coarsen.match_vertices is ops.match_vertices
assert jetpart.refine.jetlp_pass is ops.jetlp_pass
assert jetpart.rebalance.weak_rebalance_pass is ops.weak_rebalance_pass
assert jetpart.conn.build_conn is ops.build_conn
assert jetpart.initpart.initial_partition is ops.initial_partition
assert jetpart.graph.cutsize is J.cutsize
assert jetpart.errors.PreprocessError is J.PreprocessError
assert jetpart.graph.PreprocessError is J.PreprocessError
assert jetpart.driver.BalanceInfeasibleError is J.BalanceInfeasibleError
# host-side reference code is the reference's own
assert jetpart.graph.preprocess.__module__.startswith("_jetpart_reference")
print("ok")
"""


@pytest.mark.skipif(not REF.exists(), reason="reference not installed in baseline/_ref")
def test_binding_rebinds_hot_path():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [str(ROOT / "paper_2304_13194_b200" / "compat"), str(ROOT)]))
    p = subprocess.run([sys.executable, "-c", CHECK], env=env, capture_output=True, text=True,
                       timeout=120)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout + p.stderr


@pytest.mark.skipif(not REF.exists(), reason="reference not installed in baseline/_ref")
def test_cli_module_entry_resolves():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [str(ROOT / "paper_2304_13194_b200" / "compat"), str(ROOT)]))
    p = subprocess.run([sys.executable, "-m", "jetpart.cli", "--help"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and "--k" in p.stdout, p.stdout + p.stderr
