"""Pins of the oracle's SBESPAR sparsification estimator (NEXT-1; PAPER.md:1402-1438,
§Approximation by Sparsification; SPEC.md:381-435 for the test ideas).  CPU only."""
import numpy as np

import oracle as O
from synth import graphs as G


def test_generator_is_splitmix64():
    # SplitMix64 (Steele, Lea, Flood 2014; Vigna's reference splitmix64.c) from state 0: the
    # first output is 0xE220A8397B1DCDAF, a published constant
    assert O.sm64(0) == 0xE220A8397B1DCDAF


def test_rho_one_is_the_exact_count():
    g = G.random_bipartite(40, 30, 0.4, 0.6, seed=5)
    s = O.sparsify(g, 1.0, seed=9, trial=3)
    assert np.array_equal(s.row_ptr, g.row_ptr) and np.array_equal(s.col, g.col)
    assert np.array_equal(s.sign, g.sign)
    exact = O.route_g(g)["B"]
    assert O.estimate(g, 1.0, trials=3, seed=1)["estimates"] == [float(exact)] * 3


def test_retained_fraction_concentrates():
    # rho = 0.5 on a 10^4-edge graph keeps a fraction in [0.45, 0.55]
    g = G.random_bipartite(200, 100, 0.5, 0.5, seed=2)
    assert 9000 <= g.nnz <= 11000
    for t in range(3):
        s = O.sparsify(g, 0.5, seed=11, trial=t)
        assert 0.45 <= s.nnz / g.nnz <= 0.55
        # the sample is a subgraph with its signs: every kept (u, v, sign) is an input edge
        edges = set(zip(*[a.tolist() for a in g.edges()]))
        assert set(zip(*[a.tolist() for a in s.edges()])) <= edges


def test_estimator_is_unbiased_and_variance_falls_with_rho():
    # 30x30 random graph (seed 3, p_edge 0.5, p_pos 0.5), 400 trials:
    # |mean - exact| <= 3 sigma / sqrt(T); variance at rho = 0.3 >= variance at rho = 0.7
    g = G.random_bipartite(30, 30, 0.5, 0.5, seed=3)
    exact = O.route_g(g)["B"]
    assert exact >= 1000
    var = {}
    for rho in (0.3, 0.5, 0.7):
        est = np.array(O.estimate(g, rho, trials=400, seed=17)["estimates"])
        assert abs(est.mean() - exact) <= 3 * est.std(ddof=1) / np.sqrt(est.size), rho
        var[rho] = est.var(ddof=1)
    assert var[0.3] >= var[0.7]
