import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs, cutbddc as cb
for name, kw in [("cfg1", {}), ("cfg2", dict(weighting="stiffness", objects="cef")), ("cfg3", {})]:
    cfg = configs.get(name, **kw)
    o = Oracle(cfg); o.setup()
    s = cb.GpuSolver(0)
    t = time.time(); pb = cb.prepare(s, cfg); t1 = time.time()
    print(name, "prepare", t1 - t, s.stats(), flush=True)
    print(" dirichlet eq", np.array_equal(pb.dirichlet, o.dirichlet()))
    bo, bg = o.rhs(), s.rhs(); print(" rhs err", np.abs(bo - bg).max() / np.abs(bo).max())
    x = np.random.default_rng(0).uniform(-1, 1, o.n_dof)
    print(" spmv err", np.linalg.norm(o.spmv(x) - s.spmv(x)) / np.linalg.norm(o.spmv(x)))
    beo, vo = o.cells(); beg, vg = s.cells(); print(" beta err", np.abs(beo - beg).max() / max(1e-300, np.abs(beo).max()), "void eq", np.array_equal(vo, vg), "beta bitexact", np.array_equal(beo, beg))
    t = time.time(); s.setup_bddc(pb.objects, cfg.weighting); print(" setup", time.time() - t, flush=True)
    ao, ag = o.coarse_matrix(), s.coarse_matrix(); print(" coarse err", np.abs(ao - ag).max() / np.abs(ao).max())
    zo, zg = o.apply(x), s.apply(x); print(" apply err", np.linalg.norm(zo - zg) / np.linalg.norm(zo), flush=True)
    xo, ro = o.pcg(); xg, rg = s.pcg(rtol=cfg.rtol)
    print(" iters", ro["iterations"], rg["iterations"], "x err", np.linalg.norm(xo - xg) / np.linalg.norm(xo), "t_pcg", rg["t_pcg"], "lmin", rg["lmin"], flush=True)
