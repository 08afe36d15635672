"""V-degree histogram microbenchmark on config 5's col array (plain atomics vs block hash)."""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from synth import graphs as G
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhist.so"))
lib.run.restype = ctypes.c_float
g = G.make_config(5)
col = torch.from_numpy(g.col.view(np.int32)).cuda()
d = torch.zeros(g.n_v, dtype=torch.int32, device="cuda")
ref = torch.bincount(col.long(), minlength=g.n_v).int()
perm = col[torch.randperm(col.numel(), device="cuda")].contiguous()
uni = torch.randint(0, g.n_v, (col.numel(),), device="cuda", dtype=torch.int32)
for name, c in (("input", col), ("uniform", uni)):
    for var, chunk in ((0, 0), (1, 32768), (2, 32768), (2, 8192), (3, 65536), (3, 16384), (4, 8192), (4, 4096)):
        ms = lib.run(var, ctypes.c_void_p(c.data_ptr()), ctypes.c_uint64(c.numel()), ctypes.c_void_p(d.data_ptr()), g.n_v, 5, chunk)
        ok = bool(torch.equal(d, torch.bincount(c.long(), minlength=g.n_v).int()))
        print(f"{name:9s} variant {var} chunk {chunk:6d}: {ms:.3f} ms ok={ok}", flush=True)
