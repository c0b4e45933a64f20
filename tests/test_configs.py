"""BASELINE configs at full size on one GPU, inputs generated on the device
(bit-identical to the reference's generators, tests/test_generators.py):
deterministic mode must reproduce the reference's cut exactly (the reference
cut comes from the C oracle, pinned against the reference; see
tests/golden/make_quality_big.py), and the balance constraint must hold."""

import json
import math
from pathlib import Path

import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen
from paper_2304_13194_b200.driver import partition_resident

pytestmark = pytest.mark.gpu

QUALITY = json.loads((Path(__file__).parent / "golden" / "quality.json").read_text())


def _device_graph(name):
    spec = QUALITY[name]["spec"]
    if spec[0] == "rmat":
        return gen.rmat_device(spec[1], spec[2], spec[3])
    return gen.geometric_device(spec[1], spec[2], spec[3])


@pytest.mark.parametrize("name", ["rmat22", "rgg16m"])
def test_config_cut_equals_reference(name):
    if name not in QUALITY:
        pytest.skip(f"no reference cut recorded for {name}")
    case = QUALITY[name]
    dg = _device_graph(name)
    try:
        n, nnz, W = dg.info()
        assert (n, nnz // 2) == (case["n"], case["m"])
        cfg = J.RefinerConfig(k=case["k"], imbalance=case["imbalance"], seed=0, deterministic=True)
        _, pw, st = partition_resident(dg, None, cfg, want_parts=False)
        assert st.balanced
        assert int(pw.max()) <= J.part_weight_limit(W, case["k"], case["imbalance"])
        assert st.cutsize == case["cuts"]["0"]
    finally:
        dg.free()
