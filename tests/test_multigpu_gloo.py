"""Multi-GPU path on CPU: subdomain assignment and the
exchange structure of the distributed BDDC, world_size 2 over gloo.

The device path (bddc.cu) splits subdomains over ranks, keeps global dof
vectors replicated and all-reduces exactly six quantities: the stiffness
denominators (setup), the coarse matrix (setup), and per apply z0, the
coarse rhs, the weighted sum v and the harmonic correction. `_rank_apply`
restates that per-rank work in numpy with the same exchange points (the
`allreduce_sum` call sites of bddc.cu) and the test checks, on two gloo
ranks, that the exchanged result equals the single-process oracle apply —
i.e. that those six reductions are the complete data exchange.
"""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs
from paper_1703_06323_b200 import cutbddc as cb


def _morton(x, y, z):
    key = 0
    for b in range(21):
        key |= ((x >> b) & 1) << (3 * b + 2) | ((y >> b) & 1) << (3 * b + 1) | ((z >> b) & 1) << (3 * b)
    return key


@pytest.mark.parametrize("nb,world", [(2, 2), (4, 2), (4, 4), (8, 8), (6, 4), (8, 3)])
def test_assign_subdomains_contiguous_balanced(nb, world):
    block = 16
    rng = np.random.default_rng(nb * 31 + world)
    all_ids = np.arange(nb ** 3, dtype=np.int64)
    ids = np.sort(rng.choice(all_ids, size=max(world, int(0.8 * len(all_ids))), replace=False))
    r = cb.assign_subdomains(block, ids, nb * block, world)
    assert r.shape == ids.shape and r.min() == 0 and r.max() == world - 1
    counts = np.bincount(r, minlength=world)
    assert counts.max() - counts.min() <= 1, counts
    # contiguous along the Morton curve, ranks ascending
    keys = [_morton(int(b // (nb * nb)), int((b // nb) % nb), int(b % nb)) for b in ids]
    order = np.argsort(keys, kind="stable")
    assert np.all(np.diff(r[order]) >= 0)


def test_assign_subdomains_cost_weighted():
    nb, block, world = 4, 16, 2
    ids = np.arange(nb ** 3, dtype=np.int64)
    cost = np.ones(len(ids))
    cost[:8] = 20.0  # heavy subdomains
    r = cb.assign_subdomains(block, ids, nb * block, world, cost)
    loads = np.array([cost[r == k].sum() for k in range(world)])
    assert loads.max() <= loads.sum() / world + cost.max()
    assert np.bincount(r, minlength=world).min() >= 1


def test_assign_subdomains_rejects_bad_input():
    with pytest.raises(cb.CutbddcError):
        cb.assign_subdomains(16, np.zeros(0, np.int64), 64, 2)
    with pytest.raises(cb.CutbddcError):
        cb.assign_subdomains(16, np.arange(4, dtype=np.int64), 64, 0)


def _dense(sd):
    n = len(sd["l2g"])
    return sp.csr_matrix((sd["val"], sd["col"], sd["ptr"]), shape=(n, n)).toarray()


def _allreduce(a):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a, np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _rank_apply(rank, world, port, cfg_kw, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = configs.get("cfg1", **cfg_kw)
        o = Oracle(cfg, threads=2)
        o.setup()
        nd = o.n_dof
        nsd = o.info()["n_sd"]
        sds = [o.subdomain(s) for s in range(nsd)]
        block_ids = np.array([d["block_id"] for d in sds], np.int64)
        lp = cb.local_part(cfg.block, block_ids, cfg.cells, rank, world)
        local = [int(s) for s in lp.local_sd]
        ncount = np.zeros(nd, np.int64)
        for d in sds:
            ncount[d["l2g"]] += 1
        ptr, col, val = o.abar()
        abar = sp.csr_matrix((val, col, ptr), shape=(nd, nd))
        coarse = o.objects(1)
        nc = len(coarse)
        # ---- setup (local subdomains only)
        A = {s: _dense(sds[s]) for s in local}
        l2g = {s: sds[s]["l2g"] for s in local}
        dtot = np.zeros(nd)
        for s in local:
            dtot[l2g[s]] += np.diag(A[s])
        dtot = _allreduce(dtot)                                # exchange 1 (k_dtot)
        W, C, cid, K, AII, I, Phi = {}, {}, {}, {}, {}, {}, {}
        acoarse = np.zeros((nc, nc))
        for s in local:
            g = l2g[s]
            n = len(g)
            k = ncount[g]
            if cfg.weighting == configs.W_STIFFNESS:
                W[s] = np.where(k == 1, 1.0, np.diag(A[s]) / dtot[g])
            else:
                W[s] = 1.0 / k
            pos = {int(d): i for i, d in enumerate(g)}
            rows, ids = [], []
            for c, (kind, dofs, neigh) in enumerate(coarse):
                if s not in neigh:
                    continue
                row = np.zeros(n)
                for d in dofs:
                    row[pos[d]] = 1.0 if kind == configs.OBJ_C else 1.0 / len(dofs)
                rows.append(row)
                ids.append(c)
            C[s] = np.array(rows).reshape(len(rows), n)
            cid[s] = np.array(ids, np.int64)
            rho = np.mean(np.diag(A[s]))
            K[s] = A[s] + rho * C[s].T @ C[s]
            Wm = np.linalg.solve(K[s], C[s].T)
            S = C[s] @ Wm
            S = 0.5 * (S + S.T)
            Phi[s] = np.linalg.solve(S, Wm.T).T
            ac = Phi[s].T @ A[s] @ Phi[s]
            acoarse[np.ix_(cid[s], cid[s])] += 0.5 * (ac + ac.T)
            I[s] = np.flatnonzero(k == 1)
            AII[s] = A[s][np.ix_(I[s], I[s])]
        acoarse = _allreduce(acoarse)                          # exchange 2 (coarse matrix)

        # ---- apply with the device path's exchange points
        def apply(r):
            z0 = np.zeros(nd)
            for s in local:
                gi = l2g[s][I[s]]
                z0[gi] = np.linalg.solve(AII[s], r[gi])
            z0 = _allreduce(z0)                                # exchange 3 (z0)
            r1 = np.where(ncount >= 2, r - abar @ z0, 0.0)
            gc = np.zeros(nc)
            ys, cys = {}, {}
            for s in local:
                rl = W[s] * r1[l2g[s]]
                np.add.at(gc, cid[s], Phi[s].T @ rl)
                ys[s] = np.linalg.solve(K[s], rl)
                cys[s] = C[s] @ ys[s]
            gc = _allreduce(gc)                                # exchange 4 (coarse rhs)
            zc = np.linalg.solve(acoarse, gc) if nc else gc
            v = np.zeros(nd)
            for s in local:
                y = ys[s] + Phi[s] @ (zc[cid[s]] - cys[s])
                v[l2g[s]] += W[s] * y
            v = _allreduce(v)                                  # exchange 5 (weighted sum)
            av = np.where(ncount == 1, abar @ v, 0.0)
            corr = np.zeros(nd)
            for s in local:
                gi = l2g[s][I[s]]
                corr[gi] = -np.linalg.solve(AII[s], av[gi])
            corr = _allreduce(corr)                            # exchange 6 (harmonic correction)
            return z0 + v + corr

        rng = np.random.default_rng(7)
        r = rng.standard_normal(nd)
        z = apply(r)
        if rank == 0:
            zo = o.apply(r)
            ao = o.coarse_matrix()
            np.save(os.path.join(result_dir, "z.npy"), z)
            np.save(os.path.join(result_dir, "zo.npy"), zo)
            np.save(os.path.join(result_dir, "ac.npy"), acoarse)
            np.save(os.path.join(result_dir, "aco.npy"), ao)
        counts = _allreduce(np.bincount(lp.rank_of_sd, minlength=world) * (rank == 0) + 0.0)
        mine = np.zeros(nsd)
        mine[local] = 1.0
        cover = _allreduce(mine)
        if rank == 0:
            np.save(os.path.join(result_dir, "cover.npy"), cover)
            np.save(os.path.join(result_dir, "counts.npy"), counts)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kw", [dict(weighting="stiffness", objects="cef"), dict(objects="ce")])
def test_distributed_apply_world2_equals_oracle(kw, tmp_path):
    mp.spawn(_rank_apply, args=(2, _free_port(), kw, str(tmp_path)), nprocs=2, join=True)
    cover = np.load(tmp_path / "cover.npy")
    assert np.all(cover == 1.0)  # every subdomain on exactly one rank
    counts = np.load(tmp_path / "counts.npy")
    assert counts.min() >= 1
    ac, aco = np.load(tmp_path / "ac.npy"), np.load(tmp_path / "aco.npy")
    assert np.abs(ac - aco).max() <= 1e-10 * np.abs(aco).max()
    z, zo = np.load(tmp_path / "z.npy"), np.load(tmp_path / "zo.npy")
    assert np.linalg.norm(z - zo) <= 1e-9 * np.linalg.norm(zo)
