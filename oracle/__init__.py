"""CPU oracle for balanced butterfly counting (arXiv 2308.07932).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs are the only callers.  The product path (paper_2308_07932_b200)
never imports this package, and this package never imports the product path.
"""
from .oracle import (  # noqa: F401
    OracleError, build, brute, route_g, route_g_pv, Prepared, route_s, edge_brute, edge_counts, bb_base, pairs, topk_pairs, priority_order, sm64,
    sparsify, estimate, positive_subgraph, topk_vertices,
)
