"""Parity diagnostics (GPU box): for the conditioning-limited configs, compare
GPU vs oracle and oracle vs oracle-perturbed (1-ulp rho) component by
component: coarse matrix, one BDDC apply on a seeded r, PCG histories."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs
from paper_1703_06323_b200 import cutbddc as cb

CASES = [("cfg3", {}), ("cfg2", dict(weighting="topological", objects="ce")),
         ("cfg2", dict(weighting="topological", objects="cef")), ("cfg3", dict(variant="v2"))]
out = []
for name, kw in CASES:
    cfg = configs.get(name, **kw)
    os.environ.pop("ORACLE_RHO_ULPS", None)
    o = Oracle(cfg); o.setup()
    os.environ["ORACLE_RHO_ULPS"] = "1"
    op = Oracle(cfg); op.setup()
    os.environ.pop("ORACLE_RHO_ULPS", None)
    s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    ac_o, ac_p, ac_g = o.coarse_matrix(), op.coarse_matrix(), s.coarse_matrix()
    r = np.random.default_rng(5).uniform(-1, 1, o.n_dof)
    z_o, z_p, z_g = o.apply(r), op.apply(r), s.apply(r)
    xo, ro = o.pcg(); xp, rp = op.pcg(); xg, rg = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    b0 = ro["residuals"][0]
    def hist(a, b):
        n = min(len(a), len(b)); return float(np.abs(a[:n] - b[:n]).max() / b0)
    rec = dict(case=f"{name} {kw}", n_dof=o.n_dof,
               ac=dict(gpu=rel(ac_g, ac_o), ulp=rel(ac_p, ac_o)),
               apply=dict(gpu=rel(z_g, z_o), ulp=rel(z_p, z_o)),
               iters=dict(oracle=ro["iterations"], ulp=rp["iterations"], gpu=rg["iterations"]),
               hist=dict(gpu=hist(rg["residuals"], ro["residuals"]), ulp=hist(rp["residuals"], ro["residuals"])),
               x=dict(gpu=rel(xg, xo), ulp=rel(xp, xo)),
               tail=dict(oracle=(ro["residuals"][-3:] / b0).tolist(), gpu=(rg["residuals"][-3:] / b0).tolist()))
    print(json.dumps(rec), flush=True)
    out.append(rec)
    s.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/parity_probe.json", "w"), indent=1)
