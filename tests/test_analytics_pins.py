"""Pins of the oracle's case-study analytics (NEXT-2; SPEC.md:437-510
for the literal examples).  CPU only."""
import itertools

import numpy as np

import oracle as O
from synth import graphs as G


def k22(signs):
    return G.from_edges(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], signs)


def test_positive_subgraph_examples():
    # all-positive -> identical; all-negative -> edgeless; K22 with one
    # negative edge -> 3-edge path with zero butterflies
    g = k22([1, 1, 1, 1])
    p = O.positive_subgraph(g)
    assert np.array_equal(p.row_ptr, g.row_ptr) and np.array_equal(p.col, g.col)
    assert O.positive_subgraph(k22([0, 0, 0, 0])).nnz == 0
    p = O.positive_subgraph(k22([1, 1, 1, 0]))
    assert p.nnz == 3 and O.brute(p)["B"] == 0 and O.brute(p)["N"] == 0


def test_positive_butterflies_per_vertex_examples():
    # vertex with < 2 positive edges -> 0; all-positive K22 -> 1 at each vertex
    b = O.brute(O.positive_subgraph(k22([1, 1, 1, 1])))
    assert list(b["bal_u"]) == [1, 1] and list(b["bal_v"]) == [1, 1]
    g = G.from_edges(3, 3, [0, 0, 1, 1, 2, 2], [0, 1, 0, 1, 0, 1], [1, 1, 1, 1, 1, 0])
    b = O.brute(O.positive_subgraph(g))
    assert b["bal_u"][2] == 0  # U2 has one positive edge


def test_pair_collaboration_is_choose_two_of_common_positive_neighbours():
    # SPEC.md:475-477 and the sum invariant SPEC.md:491: per pair C(c,2), c = common positive
    # neighbours; summed over U pairs = total butterflies of the positive subgraph
    rng = np.random.default_rng(1)
    for seed in range(20):
        g = G.random_bipartite(9, 8, 0.5, 0.6, seed=seed)
        p = O.positive_subgraph(g)
        S = p.dense_sign()
        pm = O.brute(p, pairs=True)["pairs_u"]
        for a, b in itertools.combinations(range(g.n_u), 2):
            c = int(np.sum((S[a] > 0) & (S[b] > 0)))
            assert int(pm[a, b]) == c * (c - 1) // 2
        assert int(pm.sum()) == O.brute(p)["B"]


def test_topk_vertices_examples():
    # all-positive K22, PositiveDegree, k=2 -> two vertices with score 2, id order;
    # k larger than the side -> full ranking
    g = k22([1, 1, 1, 1])
    assert O.topk_vertices(g, 2, 0, "degree") == [(0, 2), (1, 2)]
    assert len(O.topk_vertices(g, 10, 1, "balanced")) == 2
    g = G.from_edges(3, 2, [0, 1, 1, 2, 2], [0, 0, 1, 0, 1], [1, 1, 1, 1, 1])
    assert O.topk_vertices(g, 3, 0, "degree") == [(1, 2), (2, 2), (0, 1)]
