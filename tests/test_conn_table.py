"""The reference's ConnectivityTable surface (conn.py:29-272) over the GPU
(csrc/conn.cu): contents against direct summation, exact-delta apply,
MoveList and Hierarchy contracts (moves.py:31-32, coarsen.py:33-44)."""

import numpy as np
import pytest

import paper_2304_13194_b200 as J

from helpers import brute_conn, brute_cutsize, graph_from_edges, random_graph, random_partition


def test_movelist_rejects_duplicates():
    with pytest.raises(ValueError, match="duplicate"):
        J.MoveList(np.array([1, 2, 1]), np.array([0, 0, 0]))
    with pytest.raises(ValueError, match="align"):
        J.MoveList(np.array([1, 2]), np.array([0]))


def test_hierarchy_validate_rejects_bad_maps():
    g = graph_from_edges([(0, 1), (1, 2), (2, 3)], 4)
    c = graph_from_edges([(0, 1)], 2, vertex_weights=[2, 2])
    J.Hierarchy([g, c], [np.array([0, 0, 1, 1])]).validate()
    with pytest.raises(ValueError, match="surjective"):
        J.Hierarchy([g, c], [np.array([0, 0, 0, 0])]).validate()
    with pytest.raises(ValueError, match="length"):
        J.Hierarchy([g, c], [np.array([0, 1])]).validate()


def test_partition_rejects_inconsistent_arrays():
    from paper_2304_13194_b200 import generators as gen
    g = gen.grid_graph(8, 8)
    bad = J.Graph(g.row_offsets, g.adjacency[:-3], g.edge_weights, g.vertex_weights)
    with pytest.raises(ValueError, match="adjacency"):
        J.partition(bad, J.RefinerConfig(k=2))
    bad = J.Graph(g.row_offsets, g.adjacency, g.edge_weights[:-1], g.vertex_weights)
    with pytest.raises(ValueError, match="edge_weights"):
        J.partition(bad, J.RefinerConfig(k=2))


@pytest.mark.gpu
def test_contents_match_direct_summation():
    rng = np.random.default_rng(11)
    for _ in range(15):
        g = random_graph(rng, max_weight=4)
        st = random_partition(rng, g, int(rng.integers(1, 7)))
        t = J.build_conn(g, st)
        exp = brute_conn(g, st.parts)
        for v in range(g.n):
            assert t.row_items(v) == exp[v]
            assert t.row_capacity(v) >= len(exp[v])
        rows = rng.integers(0, g.n, 50)
        ps = rng.integers(0, st.k, 50)
        got = t.get_many(rows, ps)
        assert got.tolist() == [exp[r].get(int(p), 0) for r, p in zip(rows, ps)]
        tr, tp, tw = t.nonzero_triples()
        flat = sorted((v, p, w) for v in range(g.n) for p, w in exp[v].items())
        assert list(zip(tr.tolist(), tp.tolist(), tw.tolist())) == flat


@pytest.mark.gpu
def test_star_row_and_allocation_bound():
    g = graph_from_edges([(0, i) for i in range(1, 7)], 7)
    st = J.PartitionState.from_parts(g, [0] + [3] * 6, 128)
    t = J.build_conn(g, st)
    assert t.row_items(0) == {3: 6}
    assert t.row_capacity(0) < 128
    budget = g.n + 2 * int(np.minimum(np.diff(g.row_offsets), 128).sum())
    assert t.allocated_slots <= budget + t.slack_slots


@pytest.mark.gpu
def test_apply_exact_deltas_and_errors():
    rng = np.random.default_rng(3)
    for trial in range(20):
        g = random_graph(rng, n_lo=20, n_hi=120, max_weight=5, max_vertex_weight=3)
        k = int(rng.integers(2, 9))
        st = random_partition(rng, g, k)
        t = J.build_conn(g, st)
        for _ in range(5):
            cnt = int(rng.integers(1, max(2, g.n // 2)))
            verts = rng.choice(g.n, size=cnt, replace=False)
            dests = (st.parts[verts] + rng.integers(1, k, size=cnt)) % k
            J.update_conn(t, J.MoveList(verts, dests))
            assert st.cutsize == brute_cutsize(g, st.parts)
            assert np.array_equal(st.part_weights,
                                  np.bincount(st.parts, weights=g.vertex_weights,
                                              minlength=k).astype(np.int64))
        t.check()
    g = graph_from_edges([(0, 1, 5)], 2)
    st = J.PartitionState.from_parts(g, [0, 1], 2)
    t = J.build_conn(g, st)
    with pytest.raises(AssertionError, match="current part"):
        t.apply(J.MoveList(np.array([0]), np.array([0])))
    t.apply(J.MoveList(np.array([0]), np.array([1])))
    assert st.parts.tolist() == [1, 1] and st.cutsize == 0
    assert t.row_items(1) == {1: 5}
    t.apply(J.MoveList.empty())


@pytest.mark.gpu
def test_contract_rejects_non_matching():
    g = graph_from_edges([(0, 1), (1, 2), (2, 3)], 4)
    with pytest.raises(ValueError, match="matching"):
        J.contract(g, np.array([1, 1, 3, 2]))
