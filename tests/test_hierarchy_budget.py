"""Out-of-memory hierarchies (coarsen.cuh Hierarchy): with a byte budget the
owned levels are evicted after coarsening and rebuilt on demand during
uncoarsening by re-contracting from the highest resident level. Contraction is
a deterministic function of (fine graph, matching), so a budgeted partition
must equal the unbudgeted one bit for bit -- parts, cut, part weights and
every level's statistics -- in both modes. JET_HIER_BUDGET_MB=1 evicts every
level but the one being built, so each level below the top is rebuilt."""

import os

import numpy as np
import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen

pytestmark = pytest.mark.gpu


def _run(g, cfg, budget_mb=None):
    old = os.environ.get("JET_HIER_BUDGET_MB")
    if budget_mb is None:
        os.environ.pop("JET_HIER_BUDGET_MB", None)
    else:
        os.environ["JET_HIER_BUDGET_MB"] = str(budget_mb)
    os.environ["JET_HIER_STATS"] = "1"
    try:
        return J.partition(g, cfg)
    finally:
        os.environ.pop("JET_HIER_STATS", None)
        if old is None:
            os.environ.pop("JET_HIER_BUDGET_MB", None)
        else:
            os.environ["JET_HIER_BUDGET_MB"] = old


@pytest.mark.parametrize("name,det", [("grid27_48", True), ("grid27_48", False),
                                      ("rmat16", True), ("rmat16", False)])
def test_budgeted_hierarchy_equals_resident(name, det, capfd):
    g = gen.grid27_graph(48) if name.startswith("grid") else gen.rmat_graph(16, 16, 0)
    cfg = J.RefinerConfig(k=64, imbalance=0.03, seed=0, deterministic=det)
    a = _run(g, cfg)
    capfd.readouterr()
    b = _run(g, cfg, budget_mb=1)
    err = capfd.readouterr().err
    assert "HIER rebuilt" in err, err[-2000:]
    assert a.state.cutsize == b.state.cutsize
    assert np.array_equal(a.state.parts, b.state.parts)
    assert np.array_equal(a.state.part_weights, b.state.part_weights)
    la = [(lv["n"], lv["m"], lv["iterations"], lv["cut_out"]) for lv in a.metrics["levels"]]
    lb = [(lv["n"], lv["m"], lv["iterations"], lv["cut_out"]) for lv in b.metrics["levels"]]
    assert la == lb
