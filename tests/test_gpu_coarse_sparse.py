"""Nested-dissection coarse factor (coarse_sparse.cu): the default for
n_c > 4096 (cfg5 and the multi-GPU weak-scaling meshes); CUTBDDC_COARSE=sparse
forces it on the small configurations so it is compared with the oracle here
(the exact tier of test_gpu_parity.py), and with the dense Cholesky + inverse
path on one apply."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs
from paper_1703_06323_b200 import cutbddc as cb

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,kw", [
    ("cfg2", {"weighting": "stiffness", "objects": "ce"}),
    ("cfg2", {"weighting": "stiffness", "objects": "cef"}),
    ("cfg3", {"variant": "v1"}),
    ("cfg4", {}),
])
def test_sparse_coarse_matches_oracle(monkeypatch, name, kw):
    cfg = configs.get(name, **kw)
    o = Oracle(cfg)
    o.setup()
    monkeypatch.setenv("CUTBDDC_COARSE", "sparse")
    s = cb.GpuSolver(0)
    pb = cb.prepare(s, cfg)
    s.setup_bddc(pb.objects, cfg.weighting)
    assert _rel(s.coarse_matrix(), o.coarse_matrix()) <= 1e-12
    r = np.random.default_rng(5).uniform(-1, 1, o.n_dof)
    assert _rel(s.apply(r), o.apply(r)) <= 1e-11
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    xo, repo = o.pcg()
    assert rep["iterations"] == repo["iterations"]
    assert _rel(x, xo) <= 1e-8
    res, reso = np.asarray(rep["residuals"]), np.asarray(repo["residuals"])
    assert np.abs(res - reso).max() <= 1e-8 * reso[0]
    s.close()


def test_sparse_coarse_equals_dense_coarse(monkeypatch):
    cfg = configs.get("cfg4")
    out = []
    for mode in ("dense", "sparse"):
        monkeypatch.setenv("CUTBDDC_COARSE", mode)
        s = cb.GpuSolver(0)
        pb = cb.prepare(s, cfg)
        s.setup_bddc(pb.objects, cfg.weighting)
        r = np.random.default_rng(11).uniform(-1, 1, pb.mesh.n_dof)
        out.append(s.apply(r))
        s.close()
    assert _rel(out[1], out[0]) <= 1e-12
