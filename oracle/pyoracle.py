"""ctypes harness for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU legs
(cpu_baseline and --impl reference); never by the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Cfg(C.Structure):
    _fields_ = [
        ("cells", C.c_int * 3),
        ("lo", C.c_double * 3),
        ("hi", C.c_double * 3),
        ("translation", C.c_double * 3),
        ("block", C.c_int),
        ("n_balls", C.c_int),
        ("balls", C.POINTER(C.c_double)),
        ("threads", C.c_int),
        ("problem", C.c_int),
    ]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-j8"], cwd=_HERE, check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
    return _lib


def _check(code):
    if code != 0:
        raise OracleError(code, lib().orc_last_error().decode())


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


D, I, U8, I64 = C.c_double, C.c_int, C.c_ubyte, C.c_longlong


class Oracle:
    """One problem instance: geometry + classification (+ partition/assembly
    when block > 0). Methods mirror the reference's operations."""

    def __init__(self, cfg, threads: int = 0, block: int | None = None):
        self.cfg = cfg
        L = lib()
        balls = np.ascontiguousarray(np.asarray(cfg.balls, dtype=np.float64).reshape(-1))
        c = _Cfg()
        c.cells[:] = [cfg.cells] * 3
        c.lo[:] = list(cfg.lo)
        c.hi[:] = list(cfg.hi)
        c.translation[:] = list(cfg.translation)
        c.block = cfg.block if block is None else block
        c.n_balls = len(cfg.balls)
        c.balls = _p(balls, D)
        c.threads = threads or os.cpu_count() or 1
        c.problem = getattr(cfg, "problem", 0)
        self._balls = balls
        h = C.c_void_p()
        _check(L.orc_create(C.byref(c), C.byref(h)))
        self.h = h
        self.n_cells = cfg.cells ** 3
        self.n_nodes = (cfg.cells + 1) ** 3
        info = self.info()
        self.n_dof = int(info["n_dof"])

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def info(self) -> dict:
        a = np.zeros(16, np.int64)
        _check(lib().orc_info(self.h, _p(a, I64)))
        keys = ["n_dof", "n_active", "n_cut", "n_interior_cells", "n_sd", "n_objects", "n_corner", "n_edge",
                "n_face", "n_dirichlet", "n_void_cells", "n_coarse", "sum_local_dofs", "max_local"]
        return {k: int(a[i]) for i, k in enumerate(keys)}

    def times(self) -> dict:
        t = np.zeros(4)
        lib().orc_times(self.h, _p(t, D))
        return dict(classify=t[0], assembly=t[1], setup=t[2], pcg=t[3])

    def mesh(self):
        phi = np.zeros(self.n_nodes)
        cls = np.zeros(self.n_cells, np.uint8)
        dof = np.zeros(self.n_nodes, np.int32)
        _check(lib().orc_mesh(self.h, _p(phi, D), _p(cls, U8), _p(dof, I)))
        return phi, cls, dof

    def cells(self):
        na = self.info()["n_active"]
        beta = np.zeros(na)
        void = np.zeros(na, np.uint8)
        _check(lib().orc_cells(self.h, _p(beta, D), _p(void, U8)))
        return beta, void

    def dirichlet(self):
        m = np.zeros(self.n_dof, np.uint8)
        _check(lib().orc_dirichlet(self.h, _p(m, U8)))
        return m

    def element(self, cell: int):
        k = np.zeros(64)
        f = np.zeros(8)
        beta = D()
        empty = I()
        _check(lib().orc_element(self.h, I64(cell), _p(k, D), _p(f, D), C.byref(beta), C.byref(empty)))
        return k.reshape(8, 8), f, beta.value, bool(empty.value)

    def rhs(self):
        b = np.zeros(self.n_dof)
        _check(lib().orc_rhs(self.h, _p(b, D)))
        return b

    def abar(self):
        nnz = C.c_longlong()
        _check(lib().orc_abar(self.h, None, None, None, C.byref(nnz)))
        ptr = np.zeros(self.n_dof + 1, np.int32)
        col = np.zeros(nnz.value, np.int32)
        val = np.zeros(nnz.value)
        _check(lib().orc_abar(self.h, _p(ptr, I), _p(col, I), _p(val, D), C.byref(nnz)))
        return ptr, col, val

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n_dof)
        _check(lib().orc_spmv(self.h, _p(x, D), _p(y, D)))
        return y

    def subdomain(self, s: int):
        info = np.zeros(8, np.int64)
        _check(lib().orc_subdomain_info(self.h, s, _p(info, I64)))
        n, nnz = int(info[0]), int(info[1])
        l2g = np.zeros(n, np.int32)
        ptr = np.zeros(n + 1, np.int32)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz)
        f = np.zeros(n)
        _check(lib().orc_subdomain(self.h, s, _p(l2g, I), _p(ptr, I), _p(col, I), _p(val, D), _p(f, D)))
        return dict(l2g=l2g, ptr=ptr, col=col, val=val, f=f, block=tuple(int(v) for v in info[2:5]),
                    block_id=int(info[5]))

    def local_solve(self, s: int, which: int, x):
        """Subdomain s, local dof order: which=0 -> A_II^{-1} on the interior
        dofs (others zeroed), which=1 -> K^{-1}, K = A + rho C^T C."""
        x = np.ascontiguousarray(x, np.float64).copy()
        _check(lib().orc_local_solve(self.h, s, which, _p(x, D)))
        return x

    def objects(self, which: int = 0):
        n = I()
        _check(lib().orc_objects(self.h, which, C.byref(n), None, None, None, None, None))
        no = n.value
        # generous buffers
        cap = self.n_dof * 8 + 16
        kinds = np.zeros(no, np.int32)
        dp = np.zeros(no + 1, np.int32)
        dofs = np.zeros(cap, np.int32)
        npt = np.zeros(no + 1, np.int32)
        neigh = np.zeros(cap, np.int32)
        _check(lib().orc_objects(self.h, which, C.byref(n), _p(kinds, I), _p(dp, I), _p(dofs, I), _p(npt, I),
                                 _p(neigh, I)))
        out = []
        for i in range(no):
            out.append((int(kinds[i]), dofs[dp[i]:dp[i + 1]].tolist(), neigh[npt[i]:npt[i + 1]].tolist()))
        return out

    def setup(self, objects=None, weighting=None, variant=None):
        c = self.cfg
        _check(lib().orc_setup(self.h, c.objects if objects is None else objects,
                               c.weighting if weighting is None else weighting,
                               c.variant if variant is None else variant))

    def weights(self):
        w = np.zeros(self.info()["sum_local_dofs"])
        _check(lib().orc_weights(self.h, _p(w, D)))
        return w

    def coarse_matrix(self):
        nc = self.info()["n_coarse"]
        a = np.zeros(nc * nc)
        _check(lib().orc_coarse_matrix(self.h, _p(a, D)))
        return a.reshape(nc, nc)

    def apply(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(self.n_dof)
        _check(lib().orc_apply(self.h, _p(r, D), _p(z, D)))
        return z

    def error_norms(self, x):
        """(|u_h - u|_L2, |u_h - u|_H1) of the manufactured solution."""
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(2)
        _check(lib().orc_error_norms(self.h, _p(x, D), _p(out, D)))
        return float(out[0]), float(out[1])

    def pcg(self, b=None, rtol=None, max_iter=None, precond=True):
        b = self.rhs() if b is None else np.ascontiguousarray(b, np.float64)
        rtol = self.cfg.rtol if rtol is None else rtol
        max_iter = self.cfg.max_iter if max_iter is None else max_iter
        x = np.zeros(self.n_dof)
        res = np.zeros(max_iter + 1)
        oi = np.zeros(4, np.int32)
        od = np.zeros(4)
        _check(lib().orc_pcg(self.h, _p(b, D), D(rtol), I(max_iter), I(1 if precond else 0), _p(x, D), _p(res, D),
                             _p(oi, I), _p(od, D)))
        it = int(oi[0])
        return x, dict(iterations=it, converged=bool(oi[1]), residuals=res[: it + 1].copy(), cond=float(od[0]),
                       lmin=float(od[1]), lmax=float(od[2]))


def cut_rule(phiv, full=False):
    phiv = np.ascontiguousarray(phiv, np.float64)
    vol = np.zeros((256, 4))
    surf = np.zeros((256, 7))
    cnt = np.zeros(3, np.int32)
    _check(lib().orc_cut_rule(_p(phiv, D), I(1 if full else 0), _p(vol, D), I(256), _p(surf, D), I(256), _p(cnt, I)))
    return vol[: cnt[0]].copy(), surf[: cnt[1]].copy(), int(cnt[2])


def gen_eigs_max(b, d, kernel_tol=1e-12):
    b = np.ascontiguousarray(b, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    out = D()
    _check(lib().orc_gen_eigs(_p(b, D), _p(d, D), I(b.shape[0]), D(kernel_tol), C.byref(out)))
    return out.value


def cholesky_solve(a_dense, b):
    a = np.asarray(a_dense, np.float64)
    n = a.shape[0]
    ptr, col, val = [0], [], []
    for i in range(n):
        for j in range(n):
            if a[i, j] != 0:
                col.append(j)
                val.append(a[i, j])
        ptr.append(len(col))
    ptr = np.asarray(ptr, np.int32)
    col = np.asarray(col, np.int32)
    val = np.asarray(val, np.float64)
    x = np.ascontiguousarray(b, np.float64).copy()
    _check(lib().orc_cholesky_solve(I(n), _p(ptr, I), _p(col, I), _p(val, D), _p(x, D)))
    return x


def condition_estimate(alpha, beta):
    a = np.ascontiguousarray(alpha, np.float64)
    b = np.ascontiguousarray(beta, np.float64)
    out = np.zeros(2)
    _check(lib().orc_condition_estimate(_p(a, D), _p(b, D), I(len(a)), _p(out, D)))
    return out[0], out[1]
