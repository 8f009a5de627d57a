import sys, numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla
sys.path.insert(0, "/root/repo")
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg2", weighting="stiffness", objects="cef")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
s.setup_bddc(pb.objects, cfg.weighting)
sten, mi, mp, da, sdof = s.local_system()
nsd, _, T = sten.shape
b1 = cfg.block + 1
rng = np.random.default_rng(0)
for which, mask, dadd in [(0, mi, None), (1, mp, da)]:
    x = rng.uniform(-1, 1, (nsd, T))
    y = s.local_solve(which, x).reshape(nsd, T)
    errs = []
    for sd in range(nsd):
        rows, cols, vals = [], [], []
        for u in range(T):
            ux, uy, uz = u // (b1 * b1), (u // b1) % b1, u % b1
            for k in range(27):
                vx, vy, vz = ux + k // 9 - 1, uy + (k // 3) % 3 - 1, uz + k % 3 - 1
                if min(vx, vy, vz) < 0 or max(vx, vy, vz) >= b1: continue
                v = (vx * b1 + vy) * b1 + vz
                if mask[sd, u] and mask[sd, v]:
                    val = sten[sd, k, u] + (dadd[sd, u] if (dadd is not None and k == 13) else 0.0)
                else:
                    val = 1.0 if k == 13 else 0.0
                if val != 0: rows.append(v); cols.append(u); vals.append(val)
        A = sp.csc_matrix((vals, (rows, cols)), shape=(T, T))
        ref = spla.spsolve(A, x[sd])
        e = np.linalg.norm(ref - y[sd]) / np.linalg.norm(ref)
        res = np.linalg.norm(A @ y[sd] - x[sd]) / np.linalg.norm(x[sd])
        errs.append((e, res, sd))
    errs.sort(reverse=True)
    print("which", which, "worst (relerr, resid, sd):", [(f"{a:.2e}", f"{b:.2e}", c) for a, b, c in errs[:5]])
