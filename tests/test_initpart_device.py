"""Initial partitioning on the device (initpart_dev.cu, one thread block per
restart; initpart.py:30-94): the whole deterministic pipeline with it must
equal the pipeline with the host restatement (initpart.cpp, itself pinned to
the reference by the pipeline goldens) bit for bit -- parts, cut, part
weights and every level's statistics -- across graph families and k up to
1024 (farthest-first seeding, disconnected remainders, ties)."""

import numpy as np
import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen

pytestmark = pytest.mark.gpu

CASES = [
    ("grid64x64", lambda: gen.grid_graph(64, 64), 4),
    ("grid256x256", lambda: gen.grid_graph(256, 256), 8),
    ("grid27_24", lambda: gen.grid27_graph(24), 64),
    ("rmat14", lambda: gen.rmat_graph(14, 16, 0), 64),
    ("rmat16_k1024", lambda: gen.rmat_graph(16, 16, 0), 1024),
    ("rgg14", lambda: gen.geometric_graph(1 << 14, 0.02, 0), 128),
]


@pytest.mark.parametrize("name,make,k", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("det", [True, False])
def test_device_initpart_equals_host(name, make, k, det):
    g = make()
    a = J.partition(g, J.RefinerConfig(k=k, imbalance=0.03, seed=3, deterministic=det))
    b = J.partition(g, J.RefinerConfig(k=k, imbalance=0.03, seed=3, deterministic=det,
                                       device_initial_partition=True))
    assert a.state.cutsize == b.state.cutsize
    assert np.array_equal(a.state.parts, b.state.parts)
    assert np.array_equal(a.state.part_weights, b.state.part_weights)
    la = [(L["n"], L["iterations"], L["cut_in"], L["cut_out"]) for L in a.metrics["levels"]]
    lb = [(L["n"], L["iterations"], L["cut_in"], L["cut_out"]) for L in b.metrics["levels"]]
    assert la == lb
