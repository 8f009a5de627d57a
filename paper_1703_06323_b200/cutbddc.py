"""Host-side mirror of the reference solver interface over the C ABI
(include/cutbddc.h, libcutbddc.so).

Operation names follow the reference: classify (mesh.cpp:114-169),
build_partition, classify_objects (+ split_edges_v1/v2,
SPEC.md:304-330), assemble_subassembled, build_weighting +
build_coarse_space, apply, pcg
(SPEC.md:431). Errors raise CutbddcError carrying the cutbddc_status code
(common.hpp:24-32). There is no CPU fallback: if libcutbddc.so is missing
or no CUDA device is present the calls fail.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import configs as _cfg

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcutbddc.so")
_lib = None

OK, INVALID_ARGUMENT, CONFIG, IO, SINGULAR, DEGENERATE, NOT_CONVERGED, INTERNAL = range(8)


class CutbddcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"cutbddc status {code}: {msg}")
        self.code = code


class _Opts(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world_size", C.c_int), ("nccl_id", C.c_void_p)]


class _Geometry(C.Structure):
    _fields_ = [("cells", C.c_int * 3), ("box_lo", C.c_double * 3), ("box_hi", C.c_double * 3),
                ("translation", C.c_double * 3), ("n_balls", C.c_int), ("balls", C.POINTER(C.c_double))]


class _MeshView(C.Structure):
    _fields_ = [("cells", C.c_int * 3), ("origin", C.c_double * 3), ("h", C.c_double * 3), ("n_dof", C.c_int64),
                ("phi", C.POINTER(C.c_double)), ("cls", C.POINTER(C.c_uint8)),
                ("dof_of_node", C.POINTER(C.c_int32))]


class _PartView(C.Structure):
    _fields_ = [("block", C.c_int), ("n_sd", C.c_int), ("block_ids", C.POINTER(C.c_int64))]


class _CoarseView(C.Structure):
    _fields_ = [("n_objects", C.c_int), ("kinds", C.POINTER(C.c_int32)), ("dof_ptr", C.POINTER(C.c_int64)),
                ("dofs", C.POINTER(C.c_int32)), ("neigh_ptr", C.POINTER(C.c_int64)),
                ("neigh", C.POINTER(C.c_int32))]


class _Objects(C.Structure):
    _fields_ = [("n_sd", C.c_int), ("block_ids", C.POINTER(C.c_int64)), ("n_objects", C.c_int),
                ("kinds", C.POINTER(C.c_int32)), ("dof_ptr", C.POINTER(C.c_int64)), ("dofs", C.POINTER(C.c_int32)),
                ("neigh_ptr", C.POINTER(C.c_int64)), ("neigh", C.POINTER(C.c_int32))]


class _Plan(C.Structure):
    _fields_ = [("n_loc", C.c_int64), ("n_own", C.c_int64), ("n_sd_local", C.c_int), ("n_nbr", C.c_int),
                ("loc_glob", C.POINTER(C.c_int32)), ("seg_ptr", C.POINTER(C.c_int32)),
                ("copy_ptr", C.POINTER(C.c_int32)), ("copy_src", C.POINTER(C.c_int32)), ("nbr", C.POINTER(C.c_int32)),
                ("send_ptr", C.POINTER(C.c_int64)), ("send_src", C.POINTER(C.c_int32)),
                ("recv_ptr", C.POINTER(C.c_int64))]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("cond_estimate", C.c_double),
                ("lambda_min", C.c_double), ("lambda_max", C.c_double), ("residuals", C.POINTER(C.c_double)),
                ("t_assembly", C.c_double), ("t_setup", C.c_double), ("t_pcg", C.c_double)]


EXPORTS = [
    "cutbddc_last_error", "cutbddc_gpu_create", "cutbddc_gpu_destroy", "cutbddc_gpu_classify", "cutbddc_gpu_assemble",
    "cutbddc_gpu_local_diagonals", "cutbddc_gpu_setup_bddc", "cutbddc_gpu_pcg", "cutbddc_gpu_spmv",
    "cutbddc_gpu_apply_bddc", "cutbddc_gpu_rhs", "cutbddc_gpu_coarse_matrix", "cutbddc_gpu_cells", "cutbddc_gpu_stats",
    "cutbddc_gpu_cut_elements", "cutbddc_gpu_local_system", "cutbddc_gpu_local_solve", "cutbddc_gpu_time_solves",
    "cutbddc_build_partition", "cutbddc_classify_objects", "cutbddc_objects_free", "cutbddc_gpu_classify_objects",
    "cutbddc_assign_subdomains", "cutbddc_nccl_unique_id", "cutbddc_gpu_set_distribution", "cutbddc_gpu_time_factor",
    "cutbddc_fp64_peak", "cutbddc_build_exchange_plan", "cutbddc_gpu_exchange_plan", "cutbddc_exchange_plan_free",
    "cutbddc_gpu_time_parts", "cutbddc_gpu_set_problem", "cutbddc_gpu_error_norms", "cutbddc_gpu_dense_cholesky",
    "cutbddc_host_pin", "cutbddc_host_unpin",
]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CutbddcError(INTERNAL, f"{LIB_PATH} not built (run paper_1703_06323_b200/build.py)")
        _lib = C.CDLL(LIB_PATH)
        _lib.cutbddc_last_error.restype = C.c_char_p
        _lib.cutbddc_gpu_destroy.restype = None
        _lib.cutbddc_objects_free.restype = None
        _lib.cutbddc_exchange_plan_free.restype = None
    return _lib


def _check(code: int):
    if code != 0:
        raise CutbddcError(code, lib().cutbddc_last_error().decode())


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class Mesh:
    """BackgroundMesh view (mesh.hpp:77-80): snapped node phi, cell classes,
    node -> dof map."""
    cells: int
    origin: tuple
    h: float
    phi: np.ndarray
    cls: np.ndarray
    dof_of_node: np.ndarray
    n_dof: int

    def view(self) -> _MeshView:
        v = _MeshView()
        v.cells[:] = [self.cells] * 3
        v.origin[:] = list(self.origin)
        v.h[:] = [self.h] * 3
        v.n_dof = self.n_dof
        v.phi = _p(self.phi, C.c_double)
        v.cls = _p(self.cls, C.c_uint8)
        v.dof_of_node = _p(self.dof_of_node, C.c_int32)
        return v


@dataclass
class Objects:
    """Selected coarse objects in coarse-DOF order."""
    kinds: np.ndarray
    dof_ptr: np.ndarray
    dofs: np.ndarray
    neigh_ptr: np.ndarray
    neigh: np.ndarray

    def __len__(self):
        return len(self.kinds)

    def as_list(self):
        return [(int(self.kinds[i]), self.dofs[self.dof_ptr[i]:self.dof_ptr[i + 1]].tolist(),
                 self.neigh[self.neigh_ptr[i]:self.neigh_ptr[i + 1]].tolist()) for i in range(len(self.kinds))]

    def view(self) -> _CoarseView:
        v = _CoarseView()
        v.n_objects = len(self.kinds)
        v.kinds = _p(self.kinds, C.c_int32)
        v.dof_ptr = _p(self.dof_ptr, C.c_int64)
        v.dofs = _p(self.dofs, C.c_int32)
        v.neigh_ptr = _p(self.neigh_ptr, C.c_int64)
        v.neigh = _p(self.neigh, C.c_int32)
        return v


def build_partition(mesh: Mesh, block: int) -> np.ndarray:
    n = C.c_int64()
    v = mesh.view()
    _check(lib().cutbddc_build_partition(C.byref(v), block, C.byref(n), None))
    ids = np.zeros(n.value, np.int64)
    _check(lib().cutbddc_build_partition(C.byref(v), block, C.byref(n), _p(ids, C.c_int64)))
    return ids


def classify_objects(mesh: Mesh, block: int, block_ids: np.ndarray, dirichlet: np.ndarray, objects: int,
                     variant: int = 0, local_diag: np.ndarray | None = None) -> Objects:
    v = mesh.view()
    pv = _PartView(block, len(block_ids), _p(block_ids, C.c_int64))
    out = C.POINTER(_Objects)()
    diag_p = _p(local_diag, C.c_double) if local_diag is not None else None
    dir_p = _p(dirichlet, C.c_uint8) if dirichlet is not None else None
    _check(lib().cutbddc_classify_objects(C.byref(v), C.byref(pv), dir_p, objects, variant, diag_p, C.byref(out)))
    return _take_objects(out)


def _take_objects(out) -> Objects:
    """Copy a library-owned cutbddc_objects into numpy arrays and free it."""
    o = out.contents
    no = o.n_objects
    kinds = np.ctypeslib.as_array(o.kinds, (no,)).copy() if no else np.zeros(0, np.int32)
    dptr = np.ctypeslib.as_array(o.dof_ptr, (no + 1,)).copy()
    nptr = np.ctypeslib.as_array(o.neigh_ptr, (no + 1,)).copy()
    dofs = np.ctypeslib.as_array(o.dofs, (int(dptr[-1]) + 1,))[: dptr[-1]].copy()
    neigh = np.ctypeslib.as_array(o.neigh, (int(nptr[-1]) + 1,))[: nptr[-1]].copy()
    lib().cutbddc_objects_free(out)
    return Objects(kinds.astype(np.int32), dptr, dofs.astype(np.int32), nptr, neigh.astype(np.int32))


def assign_subdomains(block: int, block_ids: np.ndarray, cells: int, world: int,
                      cost: np.ndarray | None = None) -> np.ndarray:
    """Rank of every (global) subdomain: contiguous Morton-curve chunks of
    equal estimated cost."""
    block_ids = np.ascontiguousarray(block_ids, np.int64)
    pv = _PartView(block, len(block_ids), _p(block_ids, C.c_int64))
    out = np.zeros(len(block_ids), np.int32)
    cp = _p(np.ascontiguousarray(cost, np.float64), C.c_double) if cost is not None else None
    _check(lib().cutbddc_assign_subdomains(C.byref(pv), cells, world, cp, _p(out, C.c_int32)))
    return out


def fp64_peak(device: int = 0) -> dict:
    """Measured FP64 throughput (TFLOP/s): DMMA (mma.sync m8n8k4 f64) and DFMA."""
    a, b = C.c_double(), C.c_double()
    _check(lib().cutbddc_fp64_peak(device, C.byref(a), C.byref(b)))
    return dict(dmma_tflops=a.value, dfma_tflops=b.value)


@dataclass
class ExchangePlan:
    """Interface exchange plan of one rank (include/cutbddc.h cutbddc_exchange_plan)."""
    n_loc: int
    n_own: int
    loc_glob: np.ndarray      # global dof of every local dof (segments, then ghosts)
    seg_ptr: np.ndarray       # n_sd_local + 1
    copy_ptr: np.ndarray      # n_loc + 1
    copy_src: np.ndarray      # >= 0 local slot, < 0: -1 - receive index
    nbr: np.ndarray           # neighbour ranks
    send_ptr: np.ndarray      # n_nbr + 1
    send_src: np.ndarray      # local slots of the sent values
    recv_ptr: np.ndarray      # n_nbr + 1


def _take_plan(out) -> ExchangePlan:
    p = out.contents
    nl, ns, nn = p.n_loc, p.n_sd_local, p.n_nbr
    a32 = lambda ptr, n: np.ctypeslib.as_array(ptr, shape=(max(n, 1),))[:n].copy()  # noqa: E731
    ncopy = int(p.copy_ptr[nl]) if nl else 0
    r = ExchangePlan(nl, p.n_own, a32(p.loc_glob, nl), a32(p.seg_ptr, ns + 1), a32(p.copy_ptr, nl + 1),
                     a32(p.copy_src, ncopy), a32(p.nbr, nn), a32(p.send_ptr, nn + 1),
                     np.zeros(0, np.int32), a32(p.recv_ptr, nn + 1))
    r.send_src = a32(p.send_src, int(r.send_ptr[-1]))
    lib().cutbddc_exchange_plan_free(out)
    return r


def exchange_plan(mesh: Mesh, block: int, block_ids: np.ndarray, rank_of_sd: np.ndarray, rank: int,
                  world: int) -> ExchangePlan:
    """Host-built exchange plan of `rank` (the same arrays as the device plan)."""
    block_ids = np.ascontiguousarray(block_ids, np.int64)
    ros = np.ascontiguousarray(rank_of_sd, np.int32)
    pv = _PartView(block, len(block_ids), _p(block_ids, C.c_int64))
    mv = mesh.view()
    out = C.POINTER(_Plan)()
    _check(lib().cutbddc_build_exchange_plan(C.byref(mv), C.byref(pv), _p(ros, C.c_int32), rank, world, C.byref(out)))
    return _take_plan(out)


def pin(a: np.ndarray) -> np.ndarray:
    """Page-lock a host array in place (cutbddc_host_pin): uploads from it and
    downloads into it become asynchronous DMA. Call unpin before it is freed."""
    lib().cutbddc_host_pin.argtypes = [C.c_void_p, C.c_size_t]
    _check(lib().cutbddc_host_pin(C.c_void_p(a.ctypes.data), C.c_size_t(a.nbytes)))
    return a


def unpin(a: np.ndarray) -> None:
    lib().cutbddc_host_unpin.argtypes = [C.c_void_p]
    _check(lib().cutbddc_host_unpin(C.c_void_p(a.ctypes.data)))


def nccl_unique_id() -> bytes:
    """Rank 0 creates the 128-byte NCCL id; the caller broadcasts it."""
    buf = C.create_string_buffer(128)
    _check(lib().cutbddc_nccl_unique_id(buf))
    return buf.raw


class GpuSolver:
    """One device handle: geometry -> classify -> assemble -> setup -> pcg.

    Multi-GPU: one handle per rank, created with the rank-0 NCCL id; every
    rank sets the same distribution (global partition + rank of each
    subdomain) and then assembles, sets up and solves its own subdomains;
    every call is collective over the ranks. Vectors are global-numbered
    (each rank writes the dofs it owns)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        o = _Opts(device, rank, world, C.addressof(self._id) if self._id is not None else None)
        h = C.c_void_p()
        _check(lib().cutbddc_gpu_create(C.byref(o), C.byref(h)))
        self.h = h
        self.n_dof = 0
        self.rank, self.world = rank, world

    def set_distribution(self, block: int, block_ids: np.ndarray, rank_of_sd: np.ndarray, rank: int | None = None,
                         world: int | None = None):
        """Global partition and the rank of each subdomain (every rank passes
        the same). rank/world default to the handle's; a handle without a
        communicator may take any rank's view (plan inspection only)."""
        self._bids = np.ascontiguousarray(block_ids, np.int64)
        self._ros = np.ascontiguousarray(rank_of_sd, np.int32)
        pv = _PartView(block, len(self._bids), _p(self._bids, C.c_int64))
        _check(lib().cutbddc_gpu_set_distribution(self.h, C.byref(pv), _p(self._ros, C.c_int32),
                                                  self.rank if rank is None else rank,
                                                  self.world if world is None else world))

    def set_problem(self, problem: int):
        """0: f = 1, g = 0 (BASELINE runs); 1: manufactured u = sin(5 pi |x|). Before assemble."""
        _check(lib().cutbddc_gpu_set_problem(self.h, int(problem)))

    def error_norms(self, x=None) -> tuple:
        """(|u_h - u|_L2, |u_h - u|_H1) of the manufactured problem."""
        l2, h1 = C.c_double(), C.c_double()
        xp = _p(np.ascontiguousarray(x, np.float64), C.c_double) if x is not None else None
        _check(lib().cutbddc_gpu_error_norms(self.h, xp, C.byref(l2), C.byref(h1)))
        return l2.value, h1.value

    def exchange_plan(self) -> ExchangePlan:
        """The device-built exchange plan of this handle's rank."""
        out = C.POINTER(_Plan)()
        _check(lib().cutbddc_gpu_exchange_plan(self.h, C.byref(out)))
        return _take_plan(out)

    def close(self):
        if getattr(self, "h", None):
            lib().cutbddc_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # BackgroundMesh::classify on the device
    def classify(self, cfg) -> Mesh:
        balls = np.ascontiguousarray(np.asarray(cfg.balls, np.float64).reshape(-1))
        g = _Geometry()
        g.cells[:] = [cfg.cells] * 3
        g.box_lo[:] = list(cfg.lo)
        g.box_hi[:] = list(cfg.hi)
        g.translation[:] = list(cfg.translation)
        g.n_balls = len(cfg.balls)
        g.balls = _p(balls, C.c_double)
        n = cfg.cells
        phi = np.zeros((n + 1) ** 3)
        cls = np.zeros(n ** 3, np.uint8)
        dof = np.zeros((n + 1) ** 3, np.int32)
        nd = C.c_int64()
        _check(lib().cutbddc_gpu_classify(self.h, C.byref(g), _p(phi, C.c_double), _p(cls, C.c_uint8),
                                          _p(dof, C.c_int32), C.byref(nd)))
        h = (cfg.hi[0] - cfg.lo[0]) / n
        origin = tuple(cfg.lo[d] + cfg.translation[d] for d in range(3))
        self.n_dof = nd.value
        return Mesh(n, origin, h, phi, cls, dof, nd.value)

    # assemble_subassembled on the device (block_ids: the GLOBAL partition;
    # a distributed handle assembles its own subdomains)
    def assemble(self, block: int, block_ids: np.ndarray, mesh: Mesh | None = None) -> np.ndarray:
        pv = _PartView(block, len(block_ids), _p(block_ids, C.c_int64))
        mv = mesh.view() if mesh is not None else None
        if mesh is not None:
            self.n_dof = mesh.n_dof
        dirichlet = np.zeros(self.n_dof, np.uint8)
        _check(lib().cutbddc_gpu_assemble(self.h, C.byref(mv) if mv is not None else None, C.byref(pv),
                                          _p(dirichlet, C.c_uint8)))
        return dirichlet

    def classify_objects(self, objects: int, variant: int = 0) -> Objects:
        """classify_objects (+ the v1 / v2 edge splits) on the device from the
        assembled mesh; bit-identical to the host classify_objects."""
        out = C.POINTER(_Objects)()
        _check(lib().cutbddc_gpu_classify_objects(self.h, objects, variant, C.byref(out)))
        return _take_objects(out)

    def local_diagonals(self) -> np.ndarray:
        n = C.c_int64()
        _check(lib().cutbddc_gpu_local_diagonals(self.h, None, C.byref(n)))
        d = np.zeros(n.value)
        _check(lib().cutbddc_gpu_local_diagonals(self.h, _p(d, C.c_double), C.byref(n)))
        return d

    def setup_bddc(self, objects: Objects, weighting: int):
        v = objects.view()
        _check(lib().cutbddc_gpu_setup_bddc(self.h, C.byref(v), weighting))

    def pcg(self, b=None, rtol=1e-6, max_iter=2000):
        x = np.zeros(self.n_dof)
        res = np.zeros(max_iter + 1)
        rep = _Report()
        rep.residuals = _p(res, C.c_double)
        bp = _p(np.ascontiguousarray(b, np.float64), C.c_double) if b is not None else None
        _check(lib().cutbddc_gpu_pcg(self.h, bp, _p(x, C.c_double), C.c_double(rtol), max_iter, C.byref(rep)))
        it = rep.iterations
        return x, dict(iterations=it, converged=bool(rep.converged), residuals=res[: it + 1].copy(),
                       cond=rep.cond_estimate, lmin=rep.lambda_min, lmax=rep.lambda_max, t_assembly=rep.t_assembly,
                       t_setup=rep.t_setup, t_pcg=rep.t_pcg)

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n_dof)
        _check(lib().cutbddc_gpu_spmv(self.h, _p(x, C.c_double), _p(y, C.c_double)))
        return y

    def apply(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(self.n_dof)
        _check(lib().cutbddc_gpu_apply_bddc(self.h, _p(r, C.c_double), _p(z, C.c_double)))
        return z

    def rhs(self):
        b = np.zeros(self.n_dof)
        _check(lib().cutbddc_gpu_rhs(self.h, _p(b, C.c_double)))
        return b

    def coarse_matrix(self):
        n = C.c_int()
        _check(lib().cutbddc_gpu_coarse_matrix(self.h, None, C.byref(n)))
        a = np.zeros(n.value * n.value)
        _check(lib().cutbddc_gpu_coarse_matrix(self.h, _p(a, C.c_double), C.byref(n)))
        return a.reshape(n.value, n.value)

    def cells(self):
        n = C.c_int64()
        _check(lib().cutbddc_gpu_cells(self.h, None, None, C.byref(n)))
        beta = np.zeros(n.value)
        empty = np.zeros(n.value, np.uint8)
        _check(lib().cutbddc_gpu_cells(self.h, _p(beta, C.c_double), _p(empty, C.c_uint8), C.byref(n)))
        return beta, empty

    def cut_elements(self):
        n = C.c_int64()
        _check(lib().cutbddc_gpu_cut_elements(self.h, None, None, None, C.byref(n)))
        cells = np.zeros(n.value, np.int64)
        ke = np.zeros((n.value, 8, 8))
        fe = np.zeros((n.value, 8))
        _check(lib().cutbddc_gpu_cut_elements(self.h, _p(cells, C.c_int64), _p(ke, C.c_double), _p(fe, C.c_double),
                                              C.byref(n)))
        return cells, ke, fe

    def local_system(self):
        """Slot-space test view: stencil (nsd, 27, T), interior / present masks,
        diagonal shifts and slot -> dof map."""
        st = self.stats()
        nsd, T = st["n_sd"], st["slots"]
        sten = np.zeros((nsd, 27, T))
        mi = np.zeros((nsd, T), np.uint8)
        mp = np.zeros((nsd, T), np.uint8)
        da = np.zeros((nsd, T))
        sd = np.zeros((nsd, T), np.int32)
        _check(lib().cutbddc_gpu_local_system(self.h, _p(sten, C.c_double), _p(mi, C.c_uint8), _p(mp, C.c_uint8),
                                              _p(da, C.c_double), _p(sd, C.c_int32)))
        return sten, mi, mp, da, sd

    def dense_cholesky(self, a):
        """(L, X = L^{-1}) of a dense SPD matrix by the tiled dataflow
        factorisation; CutbddcError(SINGULAR) carries .pivot on failure."""
        a = np.asfortranarray(np.asarray(a, dtype=np.float64))
        n = a.shape[0]
        l = np.zeros((n, n), np.float64, order="F")
        x = np.zeros((n, n), np.float64, order="F")
        piv = C.c_int64(-1)
        code = lib().cutbddc_gpu_dense_cholesky(self.h, n, _p(a, C.c_double), _p(l, C.c_double), _p(x, C.c_double),
                                                C.byref(piv))
        if code != OK:
            err = CutbddcError(code, lib().cutbddc_last_error().decode())
            err.pivot = piv.value
            raise err
        return np.tril(l), np.tril(x)

    def local_solve(self, which: int, x):
        x = np.ascontiguousarray(x, np.float64).copy()
        _check(lib().cutbddc_gpu_local_solve(self.h, which, _p(x, C.c_double)))
        return x

    def roofline(self, reps: int = 5):
        """Live timing of the dominant kernel family (triangular-solve sweeps
        of one BDDC apply) and its algorithmic bytes."""
        sec, byt = C.c_double(), C.c_double()
        _check(lib().cutbddc_gpu_time_solves(self.h, reps, C.byref(sec), C.byref(byt)))
        return dict(kernel="k_sweep_fwd+k_sweep_bwd (3 triangular solves of one BDDC apply)",
                    seconds=sec.value, bytes=byt.value)

    def time_parts(self, reps: int = 20) -> dict:
        """Warm device time (us) of the pieces of one PCG iteration."""
        us = np.zeros(8)
        _check(lib().cutbddc_gpu_time_parts(self.h, reps, _p(us, C.c_double)))
        keys = ["op_all", "op_interface", "op_interior", "iface_sum", "apply", "apply_solves", "spmv"]
        return {k: float(v) for k, v in zip(keys, us)}

    def factor_timing(self):
        """Device time of the last setup's numeric factorisation launch(es)
        and its flops (partial Cholesky; explicit inverse panels)."""
        sec, fc, fi = C.c_double(), C.c_double(), C.c_double()
        _check(lib().cutbddc_gpu_time_factor(self.h, C.byref(sec), C.byref(fc), C.byref(fi)))
        return dict(kernel="k_dense_dag (numeric factorisation of every front, one launch)", seconds=sec.value,
                    flops_cholesky=fc.value, flops_inverse=fi.value)

    def stats(self):
        st = np.zeros(17, np.int64)
        _check(lib().cutbddc_gpu_stats(self.h, _p(st, C.c_int64)))
        keys = ["n_dof", "n_sd", "n_coarse", "slots", "panel_total", "n_supernodes", "levels", "m_max", "n_if",
                "launches", "panel_interior", "panel_neumann", "factor_flops", "world", "has_comm", "k_corner",
                "k_shell_subdomains"]
        return {k: int(st[i]) for i, k in enumerate(keys)}


@dataclass
class Problem:
    cfg: object
    mesh: Mesh
    block_ids: np.ndarray
    dirichlet: np.ndarray
    objects: Objects


def prepare(solver: GpuSolver, cfg) -> Problem:
    """Caller side of the boundary: classify (device), partition and objects
    (host), sub-assembly (device)."""
    mesh = solver.classify(cfg)
    block_ids = build_partition(mesh, cfg.block)
    solver.set_problem(getattr(cfg, "problem", 0))
    dirichlet = solver.assemble(cfg.block, block_ids)
    diag = solver.local_diagonals() if cfg.variant == _cfg.V2 else None
    objs = classify_objects(mesh, cfg.block, block_ids, dirichlet, cfg.objects, cfg.variant, diag)
    return Problem(cfg, mesh, block_ids, dirichlet, objs)


@dataclass
class LocalPart:
    """This rank's share of the global partition."""
    rank_of_sd: np.ndarray     # per global subdomain
    local_sd: np.ndarray       # global indices of this rank's subdomains, ascending
    local_block_ids: np.ndarray


def local_part(block: int, block_ids: np.ndarray, cells: int, rank: int, world: int) -> LocalPart:
    rank_of_sd = assign_subdomains(block, block_ids, cells, world)
    local_sd = np.flatnonzero(rank_of_sd == rank).astype(np.int32)
    if len(local_sd) == 0:
        raise CutbddcError(CONFIG, f"rank {rank} received no subdomain ({len(block_ids)} subdomains, {world} ranks)")
    return LocalPart(rank_of_sd, local_sd, np.ascontiguousarray(block_ids[local_sd], np.int64))


def prepare_distributed(solver: GpuSolver, cfg) -> tuple[Problem, LocalPart]:
    """prepare() for one rank of a multi-GPU solve: the mesh, partition,
    assignment and objects are built identically on every rank (host work,
    replicated); the device work is split by subdomain."""
    if cfg.variant == _cfg.V2:
        raise CutbddcError(CONFIG, "variant v2 needs every subdomain's diagonals; not supported distributed")
    mesh = solver.classify(cfg)
    block_ids = build_partition(mesh, cfg.block)
    lp = local_part(cfg.block, block_ids, cfg.cells, solver.rank, solver.world)
    solver.set_distribution(cfg.block, block_ids, lp.rank_of_sd)
    solver.set_problem(getattr(cfg, "problem", 0))
    dirichlet = solver.assemble(cfg.block, block_ids)
    objs = classify_objects(mesh, cfg.block, block_ids, dirichlet, cfg.objects, cfg.variant, None)
    return Problem(cfg, mesh, block_ids, dirichlet, objs), lp


def solve(cfg, device: int = 0):
    """End-to-end solve of one configuration: returns (x, report, problem)."""
    s = GpuSolver(device)
    pb = prepare(s, cfg)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    return x, rep, pb, s
