import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
o = Oracle(cfg); o.setup()
s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
b = o.rhs()
x = np.zeros_like(b); r = b.copy(); z = o.apply(r); p = z.copy(); rz = r @ z
for k in range(1, 16):
    q = o.spmv(p); a = rz / (p @ q); x += a * p; r -= a * q
    zo = o.apply(r); zg = s.apply(r)
    A = o.spmv  # energy-norm error of the difference
    d = zo - zg
    print(k, "|r|/|b| %.3e" % (np.linalg.norm(r) / np.linalg.norm(b)), "apply rel2 %.3e" % (np.linalg.norm(d) / np.linalg.norm(zo)),
          "energy rel %.3e" % (np.sqrt(abs(d @ A(d))) / np.sqrt(zo @ A(zo))), "r.z rel %.3e" % (abs(r @ zo - r @ zg) / (r @ zo)))
    z = zo; rzn = r @ z; p = z + (rzn / rz) * p; rz = rzn
