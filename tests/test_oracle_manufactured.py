"""manufactured(u-case) and error_norms in the CPU
restatement: the SPEC's known answers and the paper's convergence slopes."""
import math

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs


def _u(x):
    return math.sin(5 * math.pi * math.sqrt(x[0] ** 2 + x[1] ** 2 + x[2] ** 2))


def _f(x):
    r = math.sqrt(x[0] ** 2 + x[1] ** 2 + x[2] ** 2)
    return 25 * math.pi ** 2 * math.sin(5 * math.pi * r) - 10 * math.pi * math.cos(5 * math.pi * r) / r


def test_u_at_unit_point():
    # SPEC.md:246 "u at (1,0,0) = sin(5 pi) = 0"
    assert abs(_u((1.0, 0.0, 0.0))) < 1e-14


def test_f_matches_finite_differences():
    # f cross-checked against central finite differences of u at
    # 20 random points, h_fd = 1e-5, tol 1e-6 (relative to the scale 25 pi^2)
    rng = np.random.default_rng(4)
    hf = 1e-5
    for _ in range(20):
        x = rng.uniform(0.2, 0.9, 3)
        lap = 0.0
        for d in range(3):
            e = np.zeros(3)
            e[d] = hf
            lap += (_u(x + e) - 2 * _u(x) + _u(x - e)) / hf ** 2
        assert abs(-lap - _f(x)) <= 1e-6 * 25 * math.pi ** 2 * 10  # FD truncation + round-off at h_fd = 1e-5


def _mms(cells, **kw):
    return configs.get("cfg1").with_(problem=1, cells=cells, weighting=configs.W_STIFFNESS, objects=configs.OBJ_CEF, **kw)


def test_zero_solution_norm_is_norm_of_u():
    # zero solution vs u -> L2 equals |u| by the same quadrature
    o = Oracle(_mms(20))
    l2, h1 = o.error_norms(np.zeros(o.n_dof))
    assert 0.3 < l2 < 0.4 and h1 > 5.0


@pytest.mark.slow
def test_error_convergence_slopes():
    # SPEC.md:256 / PAPER.md Fig. errorconv: L2 slope 2, H1 slope 1
    errs = []
    for n in (20, 40, 80):
        o = Oracle(_mms(n))
        o.setup()
        x, rep = o.pcg()
        assert rep["converged"]
        errs.append(o.error_norms(x))
    for (a2, a1), (b2, b1) in zip(errs, errs[1:]):
        assert 1.9 <= math.log2(a2 / b2) <= 2.1
        assert 0.95 <= math.log2(a1 / b1) <= 1.05
