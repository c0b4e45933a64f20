"""On-device generators (csrc/gen.cu) against the reference's own
rmat_graph / geometric_graph + preprocess outputs (tests/golden/generators.npz,
made by tests/golden/make_generators.py from /root/reference): bit-exact CSR."""

import numpy as np
import pytest

from paper_2304_13194_b200 import generators as gen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["rmat_a", "rmat_b", "rmat_c", "rgg_a", "rgg_b", "rgg_c"])
def test_generator_matches_reference(golden, name):
    d = golden("generators")
    args = d[name + "_args"]
    if name.startswith("rmat"):
        g = gen.rmat_graph(int(args[0]), int(args[1]), int(args[2]), tuple(d[name + "_probs"]))
    else:
        g = gen.geometric_graph(int(args[0]), float(d[name + "_radius"][0]), int(args[1]))
    assert np.array_equal(g.row_offsets, d[name + "_offs"]), name
    assert np.array_equal(g.adjacency, d[name + "_adj"].astype(np.int64)), name
    assert np.array_equal(g.edge_weights, d[name + "_ew"].astype(np.int64)), name
    assert np.array_equal(g.vertex_weights, d[name + "_vw"].astype(np.int64)), name


def test_rmat_invalid_args():
    from paper_2304_13194_b200 import _lib
    with pytest.raises(Exception):
        gen.rmat_graph(0, 8)
