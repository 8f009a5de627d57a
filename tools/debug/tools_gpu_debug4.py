import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get("cfg3")
o = Oracle(cfg); o.setup()
s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
xo, ro = o.pcg(); xg, rg = s.pcg(rtol=cfg.rtol)
a, b = ro["residuals"], rg["residuals"]
k = min(len(a), len(b))
print("iters", ro["iterations"], rg["iterations"])
print("rel hist diff", np.abs(a[:k] - b[:k]) / a[0])
print("oracle r/|b| tail", a[-3:] / a[0], "gpu", b[-3:] / b[0])
