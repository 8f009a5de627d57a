"""Oracle pinning: classification vs the reference's own code (golden
fixtures) and the paper Table counts; SPEC.md geometry/quadrature examples."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import Oracle, OracleError, cut_rule
from paper_1703_06323_b200 import configs

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "classification.json")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _case(name):
    return configs.sphere_id(int(name[-1])) if name.startswith("sphere-id") else configs.get(name)


@pytest.mark.parametrize("name", ["sphere-id1", "sphere-id2", "sphere-id3", "cfg1", "cfg2"])
def test_classification_bit_exact_vs_reference(name):
    g = GOLDEN[name]
    o = Oracle(_case(name), block=0)
    phi, cls, dof = o.mesh()
    assert o.n_dof == g["n_dof"]
    assert _sha(phi) == g["sha_phi"]
    assert _sha(cls) == g["sha_cls"]
    assert _sha(dof) == g["sha_dof_of_node"]


@pytest.mark.parametrize("k,n_el,n_dof,n_sd", [(1, 1064, 1461, 8), (2, 7160, 8577, 32), (3, 51968, 57123, 160)])
def test_paper_table_sphere_rows(k, n_el, n_dof, n_sd):
    # PAPER.md:691-695
    info = Oracle(configs.sphere_id(k)).info()
    assert (info["n_active"], info["n_dof"], info["n_sd"]) == (n_el, n_dof, n_sd)


def test_all_inside_and_all_outside():
    # SPEC.md:109-110
    c = configs.Config("in", 6, 3, [(0.5, 0.5, 0.5, 100.0)])
    o = Oracle(c, block=0)
    assert o.n_dof == 7 ** 3
    _, cls, _ = o.mesh()
    assert (cls == 0).all()
    with pytest.raises(OracleError):
        Oracle(configs.Config("out", 6, 3, [(50.0, 50.0, 50.0, 1.0)]), block=0)


def test_translation_invariance():
    # translating mesh and level set together leaves classes identical
    c = configs.get("cfg2")
    t = 0.25 * (1.0 / 40)
    c2 = c.with_(lo=(t, t, t), hi=(1 + t, 1 + t, 1 + t),
                 balls=[(b[0] + t, b[1] + t, b[2] + t, b[3]) for b in c.balls])
    _, cls1, _ = Oracle(c, block=0).mesh()
    _, cls2, _ = Oracle(c2, block=0).mesh()
    assert np.array_equal(cls1, cls2)


def test_plane_cut_quadrature():
    # unit hex, phi = x - 0.25 -> volume 0.25, area 1, normal (1,0,0)
    phiv = np.array([(l & 1) - 0.25 for l in range(8)], dtype=float)
    vol, surf, dropped = cut_rule(phiv)
    assert abs(vol[:, 3].sum() - 0.25) < 1e-12
    assert (vol[:, 3] > 0).all()
    assert abs(surf[:, 3].sum() - 1.0) < 1e-12
    assert np.allclose(surf[:, 4:7], [1, 0, 0], atol=1e-12)
    assert (vol[:, 0] <= 0.25 + 1e-14).all()
    # linear F = (x, 0, 0): int div F = vol = int_{boundary} F.n ; interface part
    # contributes 0.25 * area, the x=0 face contributes 0.
    assert abs((surf[:, 0] * surf[:, 4] * surf[:, 3]).sum() - 0.25) < 1e-12


def test_oblique_cut_divergence_theorem():
    # int_{e cap Omega} div F dV = int_{boundary} F.n for F = x e_x (div F = 1):
    # boundary = interface + cell-face pieces; on faces x=0 F.n=0, x=1 face
    # clipped analytically for a plane cut.
    a = np.array([0.3, 0.2, 0.1])
    c0 = -0.35
    phiv = np.array([a @ [(l & 1), (l >> 1) & 1, (l >> 2) & 1] + c0 for l in range(8)])
    vol, surf, _ = cut_rule(phiv)
    # interface flux of F = x e_x
    flux_if = (surf[:, 0] * surf[:, 4] * surf[:, 3]).sum()
    # x = 1 face: area of {0.3 + 0.2y + 0.1z + c0 < 0} in the unit square
    ys = np.linspace(0, 1, 2001)
    zmax = np.clip(-(0.3 + 0.2 * ys + c0) / 0.1, 0, 1)
    face = np.trapezoid(zmax, ys)
    assert abs(vol[:, 3].sum() - (flux_if + face)) < 1e-6
    assert np.allclose(np.linalg.norm(surf[:, 4:7], axis=1), 1.0, atol=1e-12)


def test_full_cell_rule():
    # SPEC.md:165-167
    vol, surf, _ = cut_rule(np.zeros(8), full=True)
    assert vol.shape[0] == 8 and surf.shape[0] == 0
    assert abs(vol[:, 3].sum() - 1) < 1e-15
    assert abs((vol[:, 3] * vol[:, 0] ** 2).sum() - 1.0 / 3.0) < 1e-14


def test_sphere_volume_converges():
    # sum eta|e| -> |Omega| at order >= 2
    errs = []
    for n in (10, 20, 40):
        c = configs.Config("s", n, n, [(0.5, 0.5, 0.5, 0.37)])
        o = Oracle(c, block=0)
        phi, cls, _ = o.mesh()
        h = 1.0 / n
        vol = 0.0
        for cell in np.nonzero(cls != 1)[0]:
            i, j, k = cell // (n * n), (cell // n) % n, cell % n
            pv = [phi[((i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)] for l in range(8)]
            if cls[cell] == 0:
                vol += h ** 3
            else:
                v, _, _ = cut_rule(np.array(pv))
                vol += v[:, 3].sum() * h ** 3
        errs.append(abs(vol - 4 / 3 * np.pi * 0.37 ** 3))
    assert errs[1] < errs[0] / 3 and errs[2] < errs[1] / 3


def test_mt19937_64_known_answer():
    rng = configs.MT19937_64()
    for _ in range(9999):
        rng()
    assert rng() == 9981545732273789042
