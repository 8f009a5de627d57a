"""Multi-GPU path on CPU: subdomain assignment, the
product's exchange plans (cutbddc_build_exchange_plan, the host twin of the
device plan in dist.cu), and the distributed BDDC + PCG over 1-4 gloo ranks.

The device path keeps one local dof space per rank (its subdomains' dofs),
sums over subdomain copies in global subdomain order with remote copies
received from neighbour ranks (one grouped send/recv per neighbour), forms
dots from per-subdomain partials gathered and added in global subdomain
order, and all-gathers the staged coarse rows / blocks. `_Rank` restates that
per-rank work in numpy driven by the product plans, and the tests check that
1, 2, 3 and 4 ranks give bit-identical results equal to the CPU oracle.
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


class _Rank:
    """One rank of the distributed solve, restated in numpy over the PRODUCT's
    exchange plan (cutbddc_build_exchange_plan: the same arrays the device
    builds, tests/test_gpu_dist.py) with the device path's exchange points
    (dist.cu / bddc.cu / pcg.cu): local dof vectors, interface sums over
    copies in global subdomain order with remote copies received from
    neighbour ranks, per-subdomain dot partials gathered and added in global
    subdomain order, staged coarse rows and blocks all-gathered."""

    def __init__(self, o, cfg, rank, world, rank_of_sd, mesh):
        self.rank, self.world = rank, world
        nsd_g = o.info()["n_sd"]
        self.sds = [o.subdomain(s) for s in range(nsd_g)]
        block_ids = np.array([d["block_id"] for d in self.sds], np.int64)
        self.plan = cb.exchange_plan(mesh, cfg.block, block_ids, rank_of_sd, rank, world)
        self.local = [int(g) for g in np.flatnonzero(rank_of_sd == rank)]
        self.nsd_g, self.ros = nsd_g, rank_of_sd
        per = np.bincount(rank_of_sd, minlength=world)
        self.maxloc = int(per.max())
        lidx = np.zeros(nsd_g, np.int64)
        for q in range(world):
            lidx[rank_of_sd == q] = np.arange(per[q])
        self.gpos = rank_of_sd.astype(np.int64) * self.maxloc + lidx
        b1 = cfg.block + 1
        self.T = b1 ** 3
        n = cfg.cells
        node_of_dof = np.zeros(mesh.n_dof, np.int64)
        nodes = np.flatnonzero(mesh.dof_of_node >= 0)
        node_of_dof[mesh.dof_of_node[nodes]] = nodes
        loc_of_glob = np.full(mesh.n_dof, -1, np.int64)
        loc_of_glob[self.plan.loc_glob] = np.arange(self.plan.n_loc)
        self.A, self.slot, self.loc, self.f = {}, {}, {}, {}
        for li, g in enumerate(self.local):
            d = self.sds[g]
            v = node_of_dof[d["l2g"]]
            i, j, k = v // ((n + 1) ** 2), (v // (n + 1)) % (n + 1), v % (n + 1)
            bi, bj, bk = d["block"]
            self.slot[g] = li * self.T + ((i - bi * cfg.block) * b1 + (j - bj * cfg.block)) * b1 + (k - bk * cfg.block)
            self.loc[g] = loc_of_glob[d["l2g"]]
            self.A[g] = _dense(d)
            self.f[g] = d["f"]
        self.ncopy = np.diff(self.plan.copy_ptr)

    # ---- exchange primitives (iface_exchange / iface_sum, gather_partials)
    def _exchange(self, Y):
        import torch
        p = self.plan
        reqs, recv = [], np.zeros(int(p.recv_ptr[-1]))
        bufs = []
        for k, q in enumerate(p.nbr):
            out = torch.from_numpy(np.ascontiguousarray(Y[p.send_src[p.send_ptr[k]:p.send_ptr[k + 1]]]))
            inn = torch.zeros(int(p.recv_ptr[k + 1] - p.recv_ptr[k]), dtype=torch.float64)
            bufs.append((k, inn))
            reqs += [dist.isend(out, int(q)), dist.irecv(inn, int(q))]
        for r in reqs:
            r.wait()
        for k, inn in bufs:
            recv[p.recv_ptr[k]:p.recv_ptr[k + 1]] = inn.numpy()
        return recv

    def isum(self, Y):
        """out[i] = Σ over the copies of local dof i (ascending global sd)."""
        recv = self._exchange(Y)
        p = self.plan
        out = np.zeros(p.n_loc)
        for i in range(p.n_loc):
            acc = 0.0
            for c in p.copy_src[p.copy_ptr[i]:p.copy_ptr[i + 1]]:
                acc += Y[c] if c >= 0 else recv[-1 - c]
            out[i] = acc
        return out

    def dot(self, a, b):
        import torch
        p = self.plan
        part = np.zeros(self.world * self.maxloc)
        for s in range(len(self.local)):
            lo, hi = p.seg_ptr[s], p.seg_ptr[s + 1]
            part[self.rank * self.maxloc + s] = float(np.dot(a[lo:hi], b[lo:hi]))
        t = torch.from_numpy(part[self.rank * self.maxloc:(self.rank + 1) * self.maxloc].copy())
        out = [torch.zeros_like(t) for _ in range(self.world)]
        dist.all_gather(out, t)
        part = torch.cat(out).numpy()
        acc = 0.0
        for g in range(self.nsd_g):
            acc += part[self.gpos[g]]
        return acc

    def gather_blocks(self, blocks):
        """every subdomain's object (an array) on every rank, by global sd"""
        out = [None] * self.world
        dist.all_gather_object(out, {g: blocks[g] for g in self.local})
        allb = {}
        for d in out:
            allb.update(d)
        return allb

    def slots(self, vec_of_sd):
        Y = np.zeros(len(self.local) * self.T)
        for g in self.local:
            Y[self.slot[g]] = vec_of_sd[g]
        return Y

    # ---- BDDC setup + apply and the PCG
    def setup(self, coarse, weighting):
        self.ncount = self.ncopy
        nc = len(coarse)
        dtot = self.isum(self.slots({g: np.diag(self.A[g]) for g in self.local}))
        self.W, self.C, self.cid, self.Phi, self.I, self.K = {}, {}, {}, {}, {}, {}
        ac = {}
        for g in self.local:
            A, loc = self.A[g], self.loc[g]
            k = self.ncount[loc]
            if weighting == configs.W_STIFFNESS:
                self.W[g] = np.where(k == 1, 1.0, np.diag(A) / dtot[loc])
            else:
                self.W[g] = 1.0 / k
            pos = {int(d): i for i, d in enumerate(self.sds[g]["l2g"])}
            rows, ids = [], []
            for c, (kind, dofs, neigh) in enumerate(coarse):
                if g not in neigh:
                    continue
                row = np.zeros(len(loc))
                for d in dofs:
                    row[pos[d]] = 1.0 if kind == configs.OBJ_C else 1.0 / len(dofs)
                rows.append(row)
                ids.append(c)
            C = np.array(rows).reshape(len(rows), len(loc))
            self.C[g], self.cid[g] = C, np.array(ids, np.int64)
            rho = np.mean(np.diag(A))
            K = A + rho * C.T @ C
            Wm = np.linalg.solve(K, C.T)
            S = C @ Wm
            S = 0.5 * (S + S.T)
            self.Phi[g] = np.linalg.solve(S, Wm.T).T
            self.K[g] = K
            a = self.Phi[g].T @ A @ self.Phi[g]
            ac[g] = 0.5 * (a + a.T)
            self.I[g] = np.flatnonzero(k == 1)
        allac = self.gather_blocks(ac)
        allcid = self.gather_blocks(self.cid)
        self.acoarse = np.zeros((nc, nc))
        for g in range(self.nsd_g):  # global subdomain order on every rank
            self.acoarse[np.ix_(allcid[g], allcid[g])] += allac[g]
        self.allcid = allcid

    def apply(self, r):
        p = self.plan
        z0 = np.zeros(p.n_loc)
        Y = np.zeros(len(self.local) * self.T)
        for g in self.local:  # interior solves, then A_GI z0 at interface slots
            loc, I = self.loc[g], self.I[g]
            zi = np.zeros(len(loc))
            zi[I] = np.linalg.solve(self.A[g][np.ix_(I, I)], r[loc[I]])
            z0[loc[I]] = zi[I]
            az = self.A[g] @ zi
            az[I] = 0.0
            Y[self.slot[g]] = az
        s_az = self.isum(Y)
        r1 = np.where(self.ncopy >= 2, r - s_az, 0.0)
        gl, ys, cys = {}, {}, {}
        for g in self.local:
            rl = self.W[g] * r1[self.loc[g]]
            gl[g] = self.Phi[g].T @ rl
            ys[g] = np.linalg.solve(self.K[g], rl)
            cys[g] = self.C[g] @ ys[g]
        allgl = self.gather_blocks(gl)
        nc = self.acoarse.shape[0]
        gc = np.zeros(nc)
        for g in range(self.nsd_g):
            gc[self.allcid[g]] += allgl[g]
        zc = np.linalg.solve(self.acoarse, gc) if nc else gc
        v = self.isum(self.slots({g: self.W[g] * (ys[g] + self.Phi[g] @ (zc[self.cid[g]] - cys[g]))
                                  for g in self.local}))
        z = z0 + v
        for g in self.local:  # harmonic correction
            loc, I = self.loc[g], self.I[g]
            av = (self.A[g] @ v[loc])[I]
            z[loc[I]] -= np.linalg.solve(self.A[g][np.ix_(I, I)], av)
        return z

    def spmv(self, x):
        return self.isum(self.slots({g: self.A[g] @ x[self.loc[g]] for g in self.local}))

    def rhs(self):
        return self.isum(self.slots(self.f))

    def pcg(self, rtol, max_iter):
        b = self.rhs()
        x, r = np.zeros_like(b), b.copy()
        hist = [np.sqrt(self.dot(b, b))]
        z = self.apply(r)
        rz = self.dot(r, z)
        p = z.copy()
        for k in range(1, max_iter + 1):
            q = self.spmv(p)
            al = rz / self.dot(p, q)
            x += al * p
            r -= al * q
            if k % 50 == 0:
                r = b - self.spmv(x)
            hist.append(np.sqrt(self.dot(r, r)))
            if hist[-1] < rtol * hist[0]:
                break
            z = self.apply(r)
            rz_new = self.dot(r, z)
            p = z + (rz_new / rz) * p
            rz = rz_new
        return x, np.array(hist)


def _cfg_small(kw):
    return configs.get("cfg1", **kw).with_(block=5)  # 64 blocks of 5^3 cells: a rich exchange topology


def _rank_main(rank, world, port, cfg_kw, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg_small(cfg_kw)
        o = Oracle(cfg, threads=1)
        o.setup()
        phi, cls, dof = o.mesh()
        mesh = cb.Mesh(cfg.cells, (0.0, 0.0, 0.0), 1.0 / cfg.cells, phi, cls, dof, o.n_dof)
        nsd = o.info()["n_sd"]
        block_ids = np.array([o.subdomain(s)["block_id"] for s in range(nsd)], np.int64)
        ros = cb.assign_subdomains(cfg.block, block_ids, cfg.cells, world)
        R = _Rank(o, cfg, rank, world, ros, mesh)
        R.setup(o.objects(1), cfg.weighting)
        rng = np.random.default_rng(7)
        rg = rng.standard_normal(o.n_dof)
        z = R.apply(rg[R.plan.loc_glob])
        x, hist = R.pcg(cfg.rtol, 200)
        own = slice(0, R.plan.n_own)
        out = dict(z=(R.plan.loc_glob[own], z[own]), x=(R.plan.loc_glob[own], x[own]), hist=hist, ac=R.acoarse)
        allout = [None] * world
        dist.all_gather_object(allout, out)
        if rank == 0:
            zg, xg = np.full(o.n_dof, np.nan), np.full(o.n_dof, np.nan)
            for d in allout:
                zg[d["z"][0]] = d["z"][1]
                xg[d["x"][0]] = d["x"][1]
            np.save(os.path.join(result_dir, f"z{world}.npy"), zg)
            np.save(os.path.join(result_dir, f"x{world}.npy"), xg)
            np.save(os.path.join(result_dir, f"hist{world}.npy"), hist)
            np.save(os.path.join(result_dir, f"ac{world}.npy"), R.acoarse)
            if world == 1:
                np.save(os.path.join(result_dir, "zo.npy"), o.apply(rg))
                xo, rep = o.pcg()
                np.save(os.path.join(result_dir, "xo.npy"), xo)
                np.save(os.path.join(result_dir, "histo.npy"), rep["residuals"])
                np.save(os.path.join(result_dir, "aco.npy"), o.coarse_matrix())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kw", [dict(weighting="stiffness", objects="cef"), dict(objects="ce")])
def test_distributed_solve_bit_identical_over_world_sizes(kw, tmp_path):
    """The distributed BDDC apply and PCG over the product's exchange plans
    on 1, 2, 3 and 4 gloo ranks: every rank count gives the same apply, the
    same residual history and the same solution BIT FOR BIT (interface sums
    in global subdomain order, dots from per-subdomain partials), and they
    match the single-process CPU oracle."""
    os.environ["OPENBLAS_NUM_THREADS"] = os.environ["OMP_NUM_THREADS"] = "1"
    for world in (1, 2, 3, 4):
        mp.spawn(_rank_main, args=(world, _free_port(), kw, str(tmp_path)), nprocs=world, join=True)
    z1, x1, h1 = (np.load(tmp_path / f"{k}1.npy") for k in ("z", "x", "hist"))
    assert not np.isnan(z1).any() and not np.isnan(x1).any()
    for world in (2, 3, 4):
        assert np.array_equal(np.load(tmp_path / f"z{world}.npy"), z1), world
        assert np.array_equal(np.load(tmp_path / f"hist{world}.npy"), h1), world
        assert np.array_equal(np.load(tmp_path / f"x{world}.npy"), x1), world
        assert np.array_equal(np.load(tmp_path / f"ac{world}.npy"), np.load(tmp_path / "ac1.npy")), world
    zo, xo, ho = np.load(tmp_path / "zo.npy"), np.load(tmp_path / "xo.npy"), np.load(tmp_path / "histo.npy")
    ac, aco = np.load(tmp_path / "ac1.npy"), np.load(tmp_path / "aco.npy")
    assert np.abs(ac - aco).max() <= 1e-10 * np.abs(aco).max()
    assert np.linalg.norm(z1 - zo) <= 1e-9 * np.linalg.norm(zo)
    # dense numpy solves vs the oracle's sparse Cholesky: the stiffness/cef
    # trajectory agrees to 1e-8; topological/ce (kappa ~ 1e3 here) amplifies
    # the solvers' rounding differences to ~1e-9 |b| late in the history
    tol = 1e-8 if kw.get("weighting") == "stiffness" else 1e-5
    assert len(h1) == len(ho) and np.abs(h1 - ho).max() <= tol * ho[0]
    assert np.linalg.norm(x1 - xo) <= tol * np.linalg.norm(xo)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exchange_plans_are_consistent(world):
    """The host exchange plans of all ranks agree with each other: message
    sizes match pairwise, every local dof's copies cover exactly its
    subdomains (ascending), every dof is owned by exactly one rank, and a
    copy value sent by one rank lands where the receiver expects it."""
    cfg = _cfg_small({})
    o = Oracle(cfg, threads=2)
    phi, cls, dof = o.mesh()
    mesh = cb.Mesh(cfg.cells, (0.0, 0.0, 0.0), 1.0 / cfg.cells, phi, cls, dof, o.n_dof)
    nsd = o.info()["n_sd"]
    sds = [o.subdomain(s) for s in range(nsd)]
    block_ids = np.array([d["block_id"] for d in sds], np.int64)
    ros = cb.assign_subdomains(cfg.block, block_ids, cfg.cells, world)
    plans = [cb.exchange_plan(mesh, cfg.block, block_ids, ros, r, world) for r in range(world)]
    owned = np.concatenate([p.loc_glob[:p.n_own] for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(o.n_dof))
    copies = {}
    for s, d in enumerate(sds):
        for gd in d["l2g"]:
            copies.setdefault(int(gd), []).append(s)
    # value of copy (sd, dof) = a unique code; each rank's slot vector carries its own copies' codes
    T = (cfg.block + 1) ** 3
    code = lambda s, gd: s * 1_000_000 + gd + 1  # noqa: E731
    slotvals = []
    for r, p in enumerate(plans):
        loc = np.flatnonzero(ros == r)
        Y = np.zeros(len(loc) * T)
        for i in range(p.n_loc):
            for c in p.copy_src[p.copy_ptr[i]:p.copy_ptr[i + 1]]:
                if c >= 0:
                    Y[c] = 1.0  # marks presence; filled below
        slotvals.append(Y)
        assert np.all(np.diff(p.copy_ptr) == [len(copies[int(gd)]) for gd in p.loc_glob])
    # fill: local copy c of local dof i belongs to the m-th local sd among its copies
    for r, p in enumerate(plans):
        for i in range(p.n_loc):
            gd = int(p.loc_glob[i])
            sd_list = copies[gd]
            for c, sdg in zip(p.copy_src[p.copy_ptr[i]:p.copy_ptr[i + 1]], sd_list):
                if c >= 0:
                    assert ros[sdg] == r
                    slotvals[r][c] = code(sdg, gd)
                else:
                    assert ros[sdg] != r
    for r, p in enumerate(plans):
        recv = np.zeros(int(p.recv_ptr[-1]))
        for k, q in enumerate(p.nbr):
            pq = plans[q]
            kk = int(np.flatnonzero(pq.nbr == r)[0])
            sent = slotvals[q][pq.send_src[pq.send_ptr[kk]:pq.send_ptr[kk + 1]]]
            assert len(sent) == p.recv_ptr[k + 1] - p.recv_ptr[k]
            recv[p.recv_ptr[k]:p.recv_ptr[k + 1]] = sent
        for i in range(p.n_loc):
            gd = int(p.loc_glob[i])
            got = [slotvals[r][c] if c >= 0 else recv[-1 - c] for c in p.copy_src[p.copy_ptr[i]:p.copy_ptr[i + 1]]]
            assert got == [code(s, gd) for s in copies[gd]], (r, gd)
