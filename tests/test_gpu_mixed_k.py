"""Mixed constrained-Neumann factor (bddc.cu):
the corner formulation K_c = A + rho C_corner^T C_corner on most subdomains
and the shell-root K = A + rho C^T C on the subdomains where K_c is singular
(a floating fragment: no corner, no Nitsche boundary; cfg5 has one). Both
give the exact constrained Neumann solve, so the preconditioner is the
oracle's whichever formulation a subdomain takes. The test hook
CUTBDDC_K_MIXED_EVERY=n puts every n-th subdomain on the shell-root K, so the
mixed path is compared with the oracle on meshes small enough to run it."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs
from paper_1703_06323_b200 import cutbddc as cb

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,kw,every", [
    ("cfg2", {"weighting": "stiffness", "objects": "ce"}, 2),
    ("cfg2", {"weighting": "stiffness", "objects": "cef"}, 3),
    ("cfg3", {"variant": "v1"}, 4),
    ("cfg4", {}, 5),
])
def test_mixed_k_matches_oracle(monkeypatch, name, kw, every):
    cfg = configs.get(name, **kw)
    o = Oracle(cfg)
    o.setup()
    monkeypatch.setenv("CUTBDDC_K_MIXED_EVERY", str(every))
    s = cb.GpuSolver(0)
    pb = cb.prepare(s, cfg)
    s.setup_bddc(pb.objects, cfg.weighting)
    st = s.stats()
    assert st["k_corner"] == 1
    assert st["k_shell_subdomains"] == (len(pb.block_ids) + every - 1) // every
    # the coarse matrix and one apply: the same operator as the oracle's
    assert _rel(s.coarse_matrix(), o.coarse_matrix()) <= 1e-12
    r = np.random.default_rng(5).uniform(-1, 1, o.n_dof)
    assert _rel(s.apply(r), o.apply(r)) <= 1e-11
    # the whole PCG (the exact tier of test_gpu_parity.py: north_star 1e-8
    # on solutions and histories)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    xo, repo = o.pcg()
    assert rep["iterations"] == repo["iterations"]
    assert _rel(x, xo) <= 1e-8
    res, reso = np.asarray(rep["residuals"]), np.asarray(repo["residuals"])
    assert np.abs(res - reso).max() <= 1e-8 * reso[0]
    s.close()


def test_mixed_k_equals_pure_formulations(monkeypatch):
    """Every subdomain on the shell-root K (n=1, still through the mixed
    path), the plain corner and the plain shell formulation: one operator."""
    cfg = configs.get("cfg2")
    r = np.random.default_rng(7).uniform(-1, 1, 0)
    out = {}
    for tag, env in (("corner", {}), ("shell", {"CUTBDDC_K_SHELL": "1"}), ("mixed1", {"CUTBDDC_K_MIXED_EVERY": "1"})):
        for k in ("CUTBDDC_K_SHELL", "CUTBDDC_K_MIXED_EVERY"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = cb.GpuSolver(0)
        pb = cb.prepare(s, cfg)
        s.setup_bddc(pb.objects, cfg.weighting)
        if r.size == 0:
            r = np.random.default_rng(7).uniform(-1, 1, pb.mesh.n_dof)
        out[tag] = (s.coarse_matrix(), s.apply(r))
        s.close()
    for tag in ("shell", "mixed1"):
        assert _rel(out[tag][0], out["corner"][0]) <= 1e-12, tag
        assert _rel(out[tag][1], out["corner"][1]) <= 1e-11, tag
