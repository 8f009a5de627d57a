import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
o = Oracle(cfg); o.setup()
s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
b = o.rhs()
def pcg(A, M, maxit=40):
    x = np.zeros_like(b); r = b.copy(); z = M(r); p = z.copy(); rz = r @ z; hist = [np.linalg.norm(b)]
    for k in range(1, maxit + 1):
        q = A(p); a = rz / (p @ q); x += a * p; r -= a * q
        if k % 50 == 0: r = b - A(x)
        hist.append(np.linalg.norm(r))
        if hist[-1] < cfg.rtol * hist[0]: break
        z = M(r); rzn = r @ z; p = z + (rzn / rz) * p; rz = rzn
    return np.array(hist)
ha = pcg(o.spmv, o.apply)
hb = pcg(o.spmv, s.apply)
hc = pcg(s.spmv, o.apply)
rng = np.random.default_rng(1)
def noisy(r):
    z = o.apply(r); return z * (1 + 1e-15 * rng.standard_normal(z.shape))
hd = pcg(o.spmv, noisy)
for name, h in [("gpuM", hb), ("gpuA", hc), ("noise1e-15", hd)]:
    k = min(len(ha), len(h))
    print(name, "iters", len(ha) - 1, len(h) - 1, "max rel diff", np.max(np.abs(ha[:k] - h[:k]) / ha[0]))
