import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2308_07932_b200 import bbf
from synth import graphs as G
for c in (3, 4, 5):
    g = G.make_config(c)
    dev = torch.device("cuda", 0)
    rp = torch.from_numpy(g.row_ptr.view(np.int64)).to(dev); col = torch.from_numpy(g.col.view(np.int32)).to(dev); sg = torch.from_numpy(g.sign).to(dev)
    outs = tuple(torch.zeros(k, dtype=torch.int64, device=dev) for k in (g.n_u, g.n_u, g.n_v, g.n_v))
    h = bbf.Graph(g.n_u, g.n_v, rp, col, sg); h.count_per_vertex(out=outs); st = h.stats(); h.free()
    print("config", c, "claimed launches per step", st["kernel_launches"], flush=True)
