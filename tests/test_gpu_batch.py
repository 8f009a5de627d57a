"""Batched solves: the translation sweep of
SPEC.md:499-507 run with several systems in flight on one GPU. Every
translated system matches the CPU oracle of the same translated mesh, and
concurrency changes nothing: the same bits as one system at a time."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import batch, configs

pytestmark = pytest.mark.gpu


def test_translation_sweep_concurrent_matches_oracle_and_sequential():
    base = configs.get("cfg2", weighting="stiffness", objects="cef")
    cfgs = batch.translation_sweep(base, 4)
    assert len({c.translation for c in cfgs}) == 4
    par, _ = batch.solve_batch(cfgs, concurrency=3)
    seq, _ = batch.solve_batch(cfgs, concurrency=1)
    for rp, rs in zip(par, seq):
        assert np.array_equal(rp.x, rs.x)
        assert np.array_equal(rp.report["residuals"], rs.report["residuals"])
    for r in par:
        o = Oracle(r.cfg)
        o.setup()
        xo, rep = o.pcg()
        assert r.n_dof == o.n_dof
        assert r.report["converged"] and r.report["iterations"] == rep["iterations"], r.cfg.translation
        assert np.abs(r.report["residuals"] - rep["residuals"]).max() <= 1e-8 * rep["residuals"][0]
        assert np.linalg.norm(r.x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_translation_sweep_v2_iteration_spread():
    """PAPER.md §5.2: the v2 coarse space keeps the iteration count nearly
    constant while the mesh slides through the body (spread <= 3)."""
    base = configs.get("cfg2", weighting="stiffness", objects="cef", variant="v2")
    res, _ = batch.solve_batch(batch.translation_sweep(base, 5), concurrency=4)
    its = [r.report["iterations"] for r in res]
    assert all(r.report["converged"] for r in res)
    assert max(its) - min(its) <= 3, its
