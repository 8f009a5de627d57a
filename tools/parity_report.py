import sys, json, numpy as np
sys.path.insert(0, "/root/repo")
from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs, cutbddc as cb
cases = [("cfg1", {}), ("cfg2", dict(weighting="topological", objects="ce")), ("cfg2", dict(weighting="topological", objects="cef")),
         ("cfg2", dict(weighting="stiffness", objects="ce")), ("cfg2", dict(weighting="stiffness", objects="cef")),
         ("cfg2", dict(weighting="stiffness", objects="cef", variant="v1")), ("cfg2", dict(weighting="stiffness", objects="cef", variant="v2")),
         ("cfg3", {}), ("cfg3", dict(variant="v2")), ("cfg3", dict(variant="v1"))]
out = []
for name, kw in cases:
    cfg = configs.get(name, **kw)
    o = Oracle(cfg); o.setup()
    s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
    xo, ro = o.pcg(); xg, rg = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    k = min(len(ro["residuals"]), len(rg["residuals"]))
    hd = float(np.abs(ro["residuals"][:k] - rg["residuals"][:k]).max() / ro["residuals"][0])
    xd = float(np.linalg.norm(xo - xg) / np.linalg.norm(xo))
    rec = dict(case=name, kw=kw, n_dof=o.n_dof, n_coarse=int(s.stats()["n_coarse"]), iters_oracle=ro["iterations"],
               iters_gpu=rg["iterations"], hist_maxdiff_rel_b=hd, x_rel=xd, cond_gpu=rg["cond"], cond_oracle=ro["cond"])
    print(json.dumps(rec), flush=True)
    out.append(rec)
    s.close()
json.dump(out, open("gpurun_out/parity_report.json", "w"), indent=1)
