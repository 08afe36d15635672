import sys, time; sys.path.insert(0, '.')
import numpy as np
from paper_2308_07932_b200 import bbf
from synth import graphs as G
g = G.config3()
with bbf.Graph.from_synth(g) as h:
    for side in (0, 1):
        t = time.time(); top = h.count_pairs_topk(100, side=side); dt = time.time() - t
        # verify each returned pair's counts exactly from the two adjacency lists
        rp = g.row_ptr.astype(np.int64)
        def nbrs(side, i):
            if side == 0:
                return dict(zip(g.col[rp[i]:rp[i+1]].tolist(), g.sign[rp[i]:rp[i+1]].tolist()))
            m = g.col == i
            us = np.repeat(np.arange(g.n_u), np.diff(rp))[m]
            return dict(zip(us.tolist(), g.sign[m].tolist()))
        ok = 0
        for (a, b, B, N) in top[:10]:
            na, nb = nbrs(side, a), nbrs(side, b)
            com = set(na) & set(nb)
            ag = sum(1 for c in com if na[c] == nb[c]); dg = len(com) - ag
            ok += (B == ag*(ag-1)//2 + dg*(dg-1)//2) and (N == ag*dg)
        print("side", side, "time %.3f s" % dt, "top1", top[0], "verified", ok, "of 10", "sorted", all(top[i][2] >= top[i+1][2] for i in range(len(top)-1)))
