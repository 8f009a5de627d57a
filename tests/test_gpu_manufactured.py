"""The manufactured problem on the GPU: the
Nitsche load vector with f = -lap u and g^D = u, the solve and the error
norms against the CPU oracle, and the discretisation error slopes."""
import math

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs
from paper_1703_06323_b200 import cutbddc as cb

pytestmark = pytest.mark.gpu


def _mms(cells):
    return configs.get("cfg1").with_(problem=1, cells=cells, weighting=configs.W_STIFFNESS, objects=configs.OBJ_CEF)


def _solve(cfg):
    s = cb.GpuSolver(0)
    pb = cb.prepare(s, cfg)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    return s, x, rep


def test_manufactured_matches_oracle():
    cfg = _mms(40)
    s, x, rep = _solve(cfg)
    o = Oracle(cfg)
    o.setup()
    b_o = o.rhs()
    assert np.abs(s.rhs() - b_o).max() <= 1e-12 * np.abs(b_o).max()
    xo, repo = o.pcg()
    assert rep["iterations"] == repo["iterations"]
    assert np.abs(rep["residuals"] - repo["residuals"]).max() <= 1e-8 * repo["residuals"][0]
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    l2, h1 = s.error_norms()
    l2o, h1o = o.error_norms(xo)
    assert abs(l2 - l2o) <= 1e-8 * l2o and abs(h1 - h1o) <= 1e-8 * h1o
    assert np.allclose(s.error_norms(x), (l2, h1), rtol=1e-12)
    s.close()


def test_error_convergence_slopes_gpu():
    errs = []
    for n in (20, 40, 80, 160):
        s, x, rep = _solve(_mms(n))
        assert rep["converged"]
        errs.append(s.error_norms())
        s.close()
    for (a2, a1), (b2, b1) in zip(errs, errs[1:]):
        assert 1.9 <= math.log2(a2 / b2) <= 2.1, errs
        assert 0.95 <= math.log2(a1 / b1) <= 1.05, errs


def test_error_norms_need_manufactured_problem():
    cfg = configs.get("cfg1")
    s, x, rep = _solve(cfg)
    with pytest.raises(cb.CutbddcError) as e:
        s.error_norms()
    assert e.value.code == cb.CONFIG
    s.close()
