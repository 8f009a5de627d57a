import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle.pyoracle import Oracle, cut_rule
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get("cfg1")
o = Oracle(cfg)
s = cb.GpuSolver(0)
m = s.classify(cfg)
phi, cls, dof = o.mesh()
print("phi equal", np.array_equal(m.phi, phi), np.abs(m.phi - phi).max())
pb = cb.prepare(s, cfg)
cells, ke, fe = s.cut_elements()
print("ncut", len(cells))
n = cfg.cells
bad = 0
for q, c in enumerate(cells[:400]):
    k, f, beta, empty = o.element(int(c))
    err = np.abs(k - ke[q]).max() / max(1e-300, np.abs(k).max())
    if err > 1e-12:
        bad += 1
        if bad <= 3:
            i, j, kk = c // (n * n), (c // n) % n, c % n
            pv = np.array([phi[((i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + kk + ((l >> 2) & 1)] for l in range(8)])
            print("cell", c, "err", err, "pv", pv)
            print(" f oracle", f, "\n f gpu", fe[q])
            vol, surf, dr = cut_rule(pv)
            print(" oracle vol sum", vol[:, 3].sum(), "nvol", len(vol), "nsurf", len(surf))
print("bad", bad)
