"""The tiled dense factorisation (dense_dag.cu: 64 x 64 tile tasks; the
diagonal tiles by the blocked POTRF + inverse, the trailing updates on DMMA)
through cutbddc_gpu_dense_cholesky, against LAPACK (numpy) on seeded SPD
matrices: every size class of the 16-column panels and 64-column tiles
(partial panels, partial tiles, several tiles), the explicit inverse, and the
pivot index of a non-positive pivot (linalg.cpp:42-54 pivot rule)."""
import numpy as np
import pytest

from paper_1703_06323_b200 import cutbddc as cb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solver():
    s = cb.GpuSolver(0)
    yield s
    s.close()


def _spd(n, seed, cond=1e3):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.geomspace(1.0, cond, n)
    return (q * ev) @ q.T


@pytest.mark.parametrize("n", [1, 2, 7, 15, 16, 17, 31, 33, 48, 63, 64, 65, 100, 128, 129, 200, 257])
def test_dense_cholesky_matches_lapack(solver, n):
    a = _spd(n, 100 + n)
    l, x = solver.dense_cholesky(a)
    l_ref = np.linalg.cholesky(a)
    assert np.linalg.norm(l - l_ref) <= 1e-12 * np.linalg.norm(l_ref)
    x_ref = np.linalg.inv(l_ref)
    assert np.linalg.norm(x - x_ref) <= 1e-11 * np.linalg.norm(x_ref)
    # backward error of the factorisation itself
    assert np.linalg.norm(l @ l.T - a) <= 1e-13 * np.linalg.norm(a)


def test_dense_cholesky_deterministic(solver):
    a = _spd(150, 7)
    l1, x1 = solver.dense_cholesky(a)
    l2, x2 = solver.dense_cholesky(a)
    assert np.array_equal(l1, l2) and np.array_equal(x1, x2)


@pytest.mark.parametrize("n,bad", [(20, 0), (20, 9), (70, 40), (130, 129)])
def test_dense_cholesky_reports_first_bad_pivot(solver, n, bad):
    """a = diag(1..) with a negative entry at `bad`: the reported pivot is the
    smallest failing index (the oracle's SparseCholesky reports the first)."""
    d = np.arange(1.0, n + 1.0)
    d[bad] = -1.0
    with pytest.raises(cb.CutbddcError) as e:
        solver.dense_cholesky(np.diag(d))
    assert e.value.code == cb.SINGULAR and e.value.pivot == bad
