import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get("cfg3")
o = Oracle(cfg); o.setup()
s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
b = o.rhs()
counts = np.zeros(o.n_dof, int)
for sd in range(o.info()["n_sd"]):
    counts[o.subdomain(sd)["l2g"]] += 1
dmask = o.dirichlet().astype(bool)
for name, r in [("b", b), ("ones", np.ones_like(b)), ("rand", np.random.default_rng(0).uniform(-1, 1, len(b)))]:
    zo, zg = o.apply(r), s.apply(r)
    d = np.abs(zo - zg)
    print(name, "rel", np.linalg.norm(zo - zg) / np.linalg.norm(zo))
    idx = np.argsort(-d)[:8]
    for i in idx:
        print("   dof", i, "zo %.6e zg %.6e diff %.2e" % (zo[i], zg[i], d[i]), "neigh", counts[i], "orphan", dmask[i])
    # error by class
    for cl, m in [("interior", counts == 1), ("interface", counts >= 2), ("orphan", dmask)]:
        if m.any(): print("   class", cl, "max diff %.2e" % d[m].max(), "max |z| %.2e" % np.abs(zo[m]).max())
