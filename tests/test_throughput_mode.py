"""Throughput mode (RefinerConfig.deterministic=False): hashed-priority
matching instead of the reference's sequential one, so partitions differ from
the reference; north_star's gate applies instead: final cutsize within 2 %
of the reference (geometric mean over seeds 0-4) and the balance constraint
always met. Reference cuts: tests/golden/quality.json (make_quality.py)."""

import json
import math
from pathlib import Path

import numpy as np
import pytest

import paper_2304_13194_b200 as J
from paper_2304_13194_b200 import generators as gen

pytestmark = pytest.mark.gpu

QUALITY = json.loads((Path(__file__).parent / "golden" / "quality.json").read_text())


def _graph(spec):
    if spec[0] == "grid":
        return gen.grid_graph(spec[1], spec[2])
    if spec[0] == "rmat":  # device generator, bit-identical to the reference's
        return gen.rmat_graph(spec[1], spec[2], spec[3])
    if spec[0] == "rgg":
        return gen.geometric_graph(spec[1], spec[2], spec[3])
    return gen.grid27_graph(spec[1])


GATED = [n for n in ("grid2d_256x256", "grid27_64", "grid27_128", "grid2d_512x512_k64",
                     "grid27_64_k256", "rmat18_k64", "rgg18_k128") if n in QUALITY]


@pytest.mark.parametrize("name", GATED)
def test_cut_within_2pct_geomean(name):
    case = QUALITY[name]
    g = _graph(case["spec"])
    k = case["k"]
    ratios = []
    for seed_s, ref_cut in case["cuts"].items():
        cfg = J.RefinerConfig(k=k, imbalance=case["imbalance"], seed=int(seed_s),
                              deterministic=False)
        res = J.partition(g, cfg)
        assert res.metrics["balanced"], (name, seed_s)
        limit = J.part_weight_limit(int(np.sum(g.vertex_weights)), k, case["imbalance"])
        assert int(res.state.part_weights.max()) <= limit
        assert res.state.cutsize == J.cutsize(g, res.state.parts)
        ratios.append(res.state.cutsize / ref_cut)
    geo = math.exp(sum(math.log(r) for r in ratios) / len(ratios))
    assert geo <= 1.02, (name, geo, ratios)


def test_throughput_matching_is_a_matching():
    g = gen.grid27_graph(24)
    from paper_2304_13194_b200 import _lib
    res = J.partition(g, J.RefinerConfig(k=16, seed=0, deterministic=False))
    assert res.metrics["balanced"]
    assert len(np.unique(res.state.parts)) == 16


@pytest.mark.parametrize("name", ["rmat22", "rgg16m"])
def test_large_configs_gate(name):
    """BASELINE configs 3-4 (device-generated, identical to the reference's
    generators) in throughput mode, partition seeds 0-4 where the reference's
    cuts are recorded (make_quality_big.py): every run balanced, cut geomean
    <= 1.02x the reference's."""
    from paper_2304_13194_b200.driver import partition_resident
    case = QUALITY[name]
    spec = case["spec"]
    dg = gen.rmat_device(spec[1], spec[2], spec[3]) if spec[0] == "rmat" else \
        gen.geometric_device(spec[1], spec[2], spec[3])
    try:
        n, _, W = dg.info()
        ratios = []
        for seed_s, ref_cut in sorted(case["cuts"].items()):
            cfg = J.RefinerConfig(k=case["k"], imbalance=case["imbalance"], seed=int(seed_s),
                                  deterministic=False)
            _, pw, st = partition_resident(dg, None, cfg, want_parts=False)
            assert st.balanced, (name, seed_s)
            assert int(pw.max()) <= J.part_weight_limit(W, case["k"], case["imbalance"])
            ratios.append(st.cutsize / ref_cut)
        geo = math.exp(sum(math.log(r) for r in ratios) / len(ratios))
        assert geo <= 1.02, (name, geo, ratios)
    finally:
        dg.free()
