"""Batched solves of many systems on one GPU.

run_translation_sweep (§5.2 "values for eps are
chosen in the closed interval [-h, +h]"): the background mesh is translated
by eps (MeshParams::translation, mesh.hpp:23) over a grid of values and every
translated system is solved. Each system is small next to a B200 (cfg4 at
64^3 keeps the triangular sweeps latency-bound at ~17% of HBM bandwidth), so
the batch runs several systems at once: one handle (one CUDA stream, its own
persistent dataflow launches and PCG graph) per worker thread, the workers
taking systems from a shared queue. The dataflow kernels never need all
their CTAs resident (tickets are taken by running CTAs only), so concurrent
launches from different handles interleave safely on the SMs.

The host side of each system (partition, objects on the device) is the same
call sequence as a single solve; ctypes releases the GIL inside the C ABI, so
the workers' host work overlaps too.
"""
from __future__ import annotations

import queue
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import configs as _cfg
from . import cutbddc as cb


def translation_sweep(cfg: _cfg.Config, n_shifts: int = 11) -> list:
    """cfg translated by eps = linspace(-h, +h, n_shifts) along (1, 1, 1)
    (the SPEC leaves the direction open; the diagonal moves every cut)."""
    h = (cfg.hi[0] - cfg.lo[0]) / cfg.cells
    eps = np.linspace(-h, h, n_shifts) if n_shifts > 1 else np.zeros(1)
    return [cfg.with_(translation=(float(e), float(e), float(e)), name=f"{cfg.name}+eps{e:+.2e}") for e in eps]


@dataclass
class BatchResult:
    cfg: _cfg.Config
    x: np.ndarray
    report: dict
    n_dof: int
    n_sd: int
    n_coarse: int


def _solve_one(s: cb.GpuSolver, cfg: _cfg.Config) -> BatchResult:
    mesh = s.classify(cfg)
    block_ids = cb.build_partition(mesh, cfg.block)
    s.assemble(cfg.block, block_ids)
    objs = s.classify_objects(cfg.objects, cfg.variant)
    s.setup_bddc(objs, cfg.weighting)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    return BatchResult(cfg, x, rep, mesh.n_dof, len(block_ids), len(objs))


class BatchRunner:
    """`concurrency` persistent handles (one stream each) and their worker
    threads; handles keep their grow-only device buffers and PCG graphs
    between systems, so a warm batch allocates nothing (cudaMalloc / cudaFree
    would synchronise the whole device and serialise the handles)."""

    def __init__(self, device: int = 0, concurrency: int = 4):
        self.solvers = [cb.GpuSolver(device) for _ in range(max(1, concurrency))]

    def run(self, cfgs: list) -> tuple[list, float]:
        """Solve every configuration; returns (results in input order, wall seconds)."""
        work: queue.Queue = queue.Queue()
        for i, c in enumerate(cfgs):
            work.put((i, c))
        out: list = [None] * len(cfgs)
        errors: list = []

        def worker(s):
            while True:
                try:
                    i, c = work.get_nowait()
                except queue.Empty:
                    return
                try:
                    out[i] = _solve_one(s, c)
                except Exception as e:  # noqa: BLE001 -- re-raised in the caller's thread
                    errors.append(e)
                    return

        t0 = time.perf_counter()
        threads = [threading.Thread(target=worker, args=(s,)) for s in self.solvers[:max(1, len(cfgs))]]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        wall = time.perf_counter() - t0
        if errors:
            raise errors[0]
        return out, wall

    def close(self):
        for s in self.solvers:
            s.close()


def solve_batch(cfgs: list, device: int = 0, concurrency: int = 4) -> tuple[list, float]:
    """One-shot batch on fresh handles (see BatchRunner for repeated batches)."""
    r = BatchRunner(device, min(concurrency, max(1, len(cfgs))))
    try:
        return r.run(cfgs)
    finally:
        r.close()
