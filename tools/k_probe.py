"""Which subdomain's corner-augmented K_c fails at a config, and what it looks
like: its constraint rows (object kinds), the failing slot, the subdomain's
present slots and how many cut cells it holds."""
import os
import sys

os.environ["CUTBDDC_K_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
s.setup_bddc(pb.objects, cfg.weighting)
print("k_corner", s.stats()["k_corner"], flush=True)
sd = int(sys.argv[2]) if len(sys.argv) > 2 else -1
if sd >= 0:
    o = pb.objects
    for i in range(len(o)):
        nb = o.neigh[o.neigh_ptr[i]:o.neigh_ptr[i + 1]]
        if sd in nb:
            print("object", i, "kind", int(o.kinds[i]), "ndofs", int(o.dof_ptr[i + 1] - o.dof_ptr[i]), "neigh", nb.tolist())
    sten, mint, mall, dadd, sdof = s.local_system()
    print("present", int(mall[sd].sum()), "interior", int(mint[sd].sum()), "corner-shifted", int((dadd[sd] != 0).sum()))

if sd >= 0:
    # dense K_c of the subdomain from its stencil + corner shifts; connected
    # components of its coupling graph and each one's smallest eigenvalue
    T = sdof.shape[1]
    b1 = round(T ** (1 / 3))
    pres = np.flatnonzero(mall[sd])
    idx = {int(t): k for k, t in enumerate(pres)}
    A = np.zeros((len(pres), len(pres)))
    for k, t in enumerate(pres):
        x, y, z = t // (b1 * b1), (t // b1) % b1, t % b1
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    u = ((x + dx) * b1 + (y + dy)) * b1 + (z + dz)
                    if 0 <= x + dx < b1 and 0 <= y + dy < b1 and 0 <= z + dz < b1 and int(u) in idx:
                        A[k, idx[int(u)]] += sten[sd, (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1), t]
    A += np.diag(dadd[sd][pres])
    G = (np.abs(A) > 0)
    comp = -np.ones(len(pres), int)
    c = 0
    for k in range(len(pres)):
        if comp[k] >= 0:
            continue
        st = [k]
        comp[k] = c
        while st:
            q = st.pop()
            for w in np.flatnonzero(G[q]):
                if comp[w] < 0:
                    comp[w] = c
                    st.append(w)
        c += 1
    print("symmetric", np.abs(A - A.T).max())
    for k in range(c):
        m = comp == k
        ev = np.linalg.eigvalsh(A[np.ix_(m, m)])
        sl = pres[m]
        print("component", k, "size", int(m.sum()), "min eig", ev[0], "max", ev[-1], "corner-shifted", int((dadd[sd][sl] != 0).sum()),
              "slots", [(int(t // (b1 * b1)), int((t // b1) % b1), int(t % b1)) for t in sl[:6]])
