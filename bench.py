"""bench.py — PCG+BDDC solved DOFs/s on B200 (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[3] ("cfg4"), the weak-scaling family at
one GPU: 64^3 background mesh, 16^3-cell subdomains, 32 seeded balls,
stiffness weighting, corner+edge+face coarse DOFs, fp64, rtol 1e-6. A "step"
is one full solve of that problem: sub-assembly (cut quadrature, beta_e,
element matrices, A^w, Abar), BDDC setup (weights, interior and constrained
Neumann factorisations, coarse basis, coarse matrix) and PCG to rtol 1e-6.

  value  = n_dof / (T_assembly + T_setup + T_pcg), device-timed (CUDA events on
           the handle's stream), mesh + partition + objects already resident.
  e2e    = the same metric through the C ABI with HOST buffers: the mesh view
           (phi, classes, dof map) and coarse objects are uploaded inside the
           timed region, the solution is read back, host object classification
           included.
  --impl reference: the CPU restatement of the reference (oracle/, the
           reference itself cannot be built: no Eigen) on the host cores.

The factor panels (~2-3 GB for cfg4) exceed the 126 MB L2, so no explicit L2
flush is needed between steps (config.l2 = "inputs larger than L2").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1703_06323_b200 import configs  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in-process
    through NVML every 20 ms (spawning nvidia-smi takes driver locks and
    stalls the solver's own host-side steps); nvidia-smi only as a fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []  # (sm_mhz, max_mhz, {reason names})
        self._stop = threading.Event()
        self._t = None

    def _nvml_sampler(self):
        import pynvml
        pynvml.nvmlInit()
        idx = self.gpu
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                idx = int(vis.split(",")[self.gpu])
            except (ValueError, IndexError):
                pass
        h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        bits = [(n, getattr(pynvml, a)) for n, a in self.REASONS]

        def sample():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            ev = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            return float(sm), float(mx), {n for n, b in bits if ev & b}
        return sample

    def _smi_sampler(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

        def sample():
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True, timeout=5).stdout.strip()
            v = [x.strip() for x in out.split(",")]
            return float(v[0]), float(v[1]), {n for (n, _), x in zip(self.REASONS, v[2:]) if x == "Active"}
        return sample

    def start(self):
        try:
            sample, period = self._nvml_sampler(), 0.02
        except Exception:
            sample, period = self._smi_sampler(), 0.2

        def run():
            while True:
                try:
                    self.rows.append(sample())
                except Exception:
                    pass
                if self._stop.wait(period):
                    break

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*(r[2] for r in self.rows))), "samples": len(self.rows)}


def cpu_reference(cfg, steps: int, warmup: int, threads: int):
    """Time the CPU restatement (oracle) of the same solve on the host cores."""
    from oracle.pyoracle import Oracle
    times = []
    info = None
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        o = Oracle(cfg, threads=threads)
        o.setup()
        x, rep = o.pcg()
        dt = time.perf_counter() - t0
        info = (o.n_dof, rep["iterations"])
        if it >= warmup:
            times.append(dt)
        del o
    return info[0], info[1], times


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n_dof, iters, times = cpu_reference(cfg, args.steps, args.warmup, threads)
    tot = sum(times)
    value = n_dof * len(times) / tot
    line = {
        "impl": "reference", "metric": "PCG+BDDC solved DOFs/sec to rtol 1e-6 (fp64)", "value": value,
        "unit": "DOF/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic (seeded ball-union geometry, BASELINE.json configs[{int(cfg.name[3:]) - 1}])",
        "config": _config(cfg, args),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": "port",
                         "sample": f"{len(times)} full solves (assembly+setup+PCG, {iters} PCG iterations) of "
                                   f"{cfg.name} {cfg.cells}^3 by the CPU restatement (oracle/, the reference "
                                   f"cannot build without Eigen)"},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(cfg, args):
    idx = int(cfg.name[3:]) - 1
    what = "weak-scaling family at " + f"{args.gpus} GPU" if cfg.name == "cfg4" else "single-GPU run"
    return {"workload": f"{cfg.name}-{cfg.cells}^3 (BASELINE.json configs[{idx}], {what})", "cells": cfg.cells, "block": cfg.block, "balls": len(cfg.balls),
            "objects": ["c", "ce", "cef"][cfg.objects], "weighting": ["topological", "stiffness"][cfg.weighting],
            "variant": ["standard", "v1", "v2"][cfg.variant], "rtol": cfg.rtol, "parallelism": f"subdomains x{args.gpus}",
            "l2": "inputs larger than L2 (factor panels > 126 MB)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank, world, local = _env_rank()
    cfg = configs.get(args.workload, gpus=max(1, args.gpus) if args.workload == "cfg4" else 1,
                      variant=args.variant)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    from paper_1703_06323_b200 import cutbddc as cb
    if world > 1:
        # gloo carries only the NCCL id and the max-over-ranks timing; the
        # solver's own exchanges run over its NCCL communicator
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        box = [cb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        solver = cb.GpuSolver(local, rank, world, box[0])
        # caller side (untimed): classify on device, partition + objects on
        # host (replicated), this rank's subdomains assembled on its GPU
        pb, lp = cb.prepare_distributed(solver, cfg)
        asm_ids = lp.local_block_ids
    else:
        solver = cb.GpuSolver(local)
        pb = cb.prepare(solver, cfg)
        lp, asm_ids = None, pb.block_ids
    mesh, block_ids, objs = pb.mesh, pb.block_ids, pb.objects
    n_dof = mesh.n_dof

    def assemble(mesh_view=None):
        d = solver.assemble(cfg.block, asm_ids, mesh=mesh_view)
        if lp is not None:
            solver.set_global_ids(len(block_ids), lp.local_sd)
        return d

    def step_device():
        assemble()                                      # mesh resident on the device
        solver.setup_bddc(objs, cfg.weighting)
        x, rep = solver.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
        return rep

    def step_e2e():
        t0 = time.perf_counter()
        dirichlet = assemble(mesh)                                     # H2D of the mesh view
        if cfg.variant == configs.V_STANDARD:                         # objects on the device
            o2 = solver.classify_objects(cfg.objects, cfg.variant)
        else:                                                          # v1/v2 edge splits: host
            diag = solver.local_diagonals() if cfg.variant == configs.V2 else None
            o2 = cb.classify_objects(mesh, cfg.block, block_ids, dirichlet, cfg.objects, cfg.variant, diag)
        solver.setup_bddc(o2, cfg.weighting)
        x, rep = solver.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)     # D2H of x
        return time.perf_counter() - t0, rep

    for _ in range(args.warmup):
        rep = step_device()
    if world > 1:
        dist.barrier()
    launches0 = solver.stats()["launches"]
    sampler = ClockSampler(local)
    sampler.start()
    dev_times, reps = [], []
    for _ in range(args.steps):
        rep = step_device()
        dev_times.append(rep["t_assembly"] + rep["t_setup"] + rep["t_pcg"])
        reps.append(rep)
    clocks = sampler.stop()
    launches = (solver.stats()["launches"] - launches0) / args.steps
    tot = max(sum(dev_times), 1e-12)
    if world > 1:
        import torch
        t = torch.tensor([tot], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    # one global problem per step, solved cooperatively by all ranks
    value = n_dof * args.steps / tot

    # e2e through the C ABI with host buffers
    for _ in range(1):
        step_e2e()
    # median of 5 wall-clock solves: one host hiccup (GC, page faults) in a
    # ~20 ms solve must not decide the number
    e2e_t = sorted(step_e2e()[0] for _ in range(5))
    e2e_mean = e2e_t[len(e2e_t) // 2]
    if world > 1:
        import torch
        t = torch.tensor([e2e_mean], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean = float(t.item())
    e2e = n_dof / e2e_mean
    n = cfg.cells
    h2d = (n + 1) ** 3 * (8 + 4) + n ** 3 + 8 * len(block_ids) + objs.dofs.nbytes + objs.neigh.nbytes + \
        objs.kinds.nbytes + objs.dof_ptr.nbytes + objs.neigh_ptr.nbytes
    d2h = 8 * n_dof + n_dof  # solution + dirichlet mask

    # roofline of the dominant kernel family (triangular solves), timed live
    rf = solver.roofline()
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved = rf["bytes"] / rf["seconds"] / 1e9 if rf["seconds"] > 0 else 0.0
    roof = {"bound": "hbm", "kernel": rf["kernel"], "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "bytes_per_launch": rf["bytes"],
            "launch_ms": 1e3 * rf["seconds"], "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"
            if peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"}
    # roofline.traffic: DRAM bytes of the same 7 sweep launches of one apply
    # from the committed ncu --set full capture (tools/ncu_traffic.py)
    tj = os.path.join(ROOT, "profiles", "r01_sweep_traffic_cfg4.json")
    if os.path.exists(tj) and world == 1 and cfg.name == "cfg4" and cfg.cells == 64:
        roof["traffic"] = json.load(open(tj))["traffic_bytes_per_apply"]
        roof["traffic_source"] = "profiles/r01_sweep_traffic_cfg4.json (ncu --set full, dram read+write)"

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cn, citers, ctimes = cpu_reference(cfg, 1, 0, threads)
        cpu = {"value": cn / ctimes[0], "unit": "DOF/s", "cores": threads, "kind": "port",
               "sample": f"1 full solve (assembly+setup+PCG, {citers} iterations) of {cfg.name} {cfg.cells}^3 by the "
                         f"CPU restatement (oracle/), {threads} threads"}
    if rank == 0:
        r0 = reps[-1]
        line = {
            "metric": "PCG+BDDC solved DOFs/sec to rtol 1e-6 (fp64)", "value": value, "unit": "DOF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded ball-union geometry, BASELINE.json configs[{int(cfg.name[3:]) - 1}])",
            "config": _config(cfg, args),
            "n_dof": n_dof, "iterations": r0["iterations"], "cond_estimate": r0["cond"],
            "phases_ms": {"assembly": 1e3 * np.mean([r["t_assembly"] for r in reps]),
                          "setup": 1e3 * np.mean([r["t_setup"] for r in reps]),
                          "pcg": 1e3 * np.mean([r["t_pcg"] for r in reps])},
            "pcg_dofs_per_s": n_dof / np.mean([r["t_pcg"] for r in reps]),
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "DOF/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "stat": "median of 5 solves", "samples_ms": [round(1e3 * t, 3) for t in e2e_t]},
            "gpu_launches": int(launches), "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
