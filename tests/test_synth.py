"""Generator checks (synth/graphs.py): determinism, sizes, simple graphs, and that the torch-CUDA
accelerated primitives reproduce the numpy recipe bit for bit."""
import os

import numpy as np
import pytest

from synth import graphs as G

GOLD = os.path.join(os.path.dirname(__file__), "golden", "synth_sha256.txt")


def golden():
    out = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        c, sha, n_u, n_v, nnz = line.split()
        out[int(c)] = (sha, int(n_u), int(n_v), int(nnz))
    return out


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_small_configs_match_recorded_hash(cfg):
    g = G.make_config(cfg)
    sha, n_u, n_v, nnz = golden()[cfg]
    assert (g.n_u, g.n_v, g.nnz) == (n_u, n_v, nnz)
    assert g.sha256() == sha


def test_config_shapes_and_simplicity():
    g = G.config1()
    assert g.nnz == 2000 and g.row_ptr[-1] == 2000
    g = G.config2()
    deg_u = np.diff(g.row_ptr.astype(np.int64))
    assert deg_u.max() <= 80
    # signs are per movie (all edges of a movie share the sign)
    u, v, s = g.edges()
    for j in np.unique(v)[:200]:
        assert len(set(s[v == j].tolist())) == 1
    for g in (G.config1(), G.config2(), G.random_bipartite(9, 7, 0.5, 0.5, 3)):
        u, v, s = g.edges()
        key = u * g.n_v + v
        assert np.unique(key).size == key.size
        assert set(np.unique(s).tolist()) <= {0, 1}


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [3, 6])
def test_large_configs_match_recorded_hash(cfg):
    g = G.make_config(cfg)
    sha, n_u, n_v, nnz = golden()[cfg]
    assert (g.n_u, g.n_v, g.nnz) == (n_u, n_v, nnz)
    assert g.sha256() == sha


@pytest.mark.gpu
def test_gpu_accelerated_generator_reproduces_numpy():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    for cfg in (3, 5, 6):
        g = G.make_config(cfg)
        assert g.sha256() == golden()[cfg][0], cfg
