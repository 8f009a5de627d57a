"""bench.py — PCG+BDDC solved DOFs/s on B200 (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[3] ("cfg4"), the weak-scaling family at
one GPU: 64^3 background mesh, 16^3-cell subdomains, 32 seeded balls,
stiffness weighting, corner+edge+face coarse DOFs, fp64, rtol 1e-6. A "step"
is one full solve of that problem: sub-assembly (cut quadrature, beta_e,
element matrices, A^w, Abar), BDDC setup (weights, interior and constrained
Neumann factorisations, coarse basis, coarse matrix) and PCG to rtol 1e-6.

  value  = n_dof / (T_assembly + T_setup + T_pcg), device-timed (CUDA events on
           the handle's stream), mesh + partition + objects already resident.
           Every timed step rebuilds the factorisation task list
           (CUTBDDC_NO_PLAN_CACHE=1): nothing computed for one step's
           geometry is reused by the next except allocations and the ND
           templates (functions of the block size only). "warm" repeats the
           measurement with the task-list cache on (the repeated-solve case).
  e2e    = the same metric through the C ABI with HOST buffers: the mesh view
           (phi, classes, dof map) uploaded, objects classified, setup, PCG,
           the solution read back; wall clock, median of 5, plan cache off.
           "e2e_fresh_handle" adds creating the handle (stream, every device
           allocation) to each solve.
  roofline       = the dominant PCG kernel family (triangular-solve sweeps),
                   HBM-bound; roofline_fp64 = the numeric factorisation
                   (k_dense_dag) against the FP64 tensor (DMMA) peak measured
                   in the same run by a committed microbenchmark (peak.cu).
  cfg5   = BASELINE.json configs[4] (256^3, ~2.9M dofs) on the same GPU: the
           only L2-busting config, where the sweep HBM fraction is the
           kernels' own streaming efficiency.
  --impl reference: the CPU restatement of the reference (oracle/, the
           reference itself cannot be built: no Eigen) on the host cores.
  --gpus N without an external launcher re-launches itself under
           torch.distributed.run with N ranks (one per GPU).

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

        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)  # constant: asked once

        def sample():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
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
            sample, period = self._nvml_sampler(), getattr(self, "period", 0.02)
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


def _relaunch(args) -> int:
    """--gpus N > 1 without torchrun: run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def _max_over_ranks(v: float, world: int) -> float:
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _time_steps(step, steps):
    reps = []
    for _ in range(steps):
        reps.append(step())
    tot = sum(r["t_assembly"] + r["t_setup"] + r["t_pcg"] for r in reps)
    return max(tot, 1e-12), reps


def _phases(reps):
    return {"assembly": 1e3 * float(np.mean([r["t_assembly"] for r in reps])),
            "setup": 1e3 * float(np.mean([r["t_setup"] for r in reps])),
            "pcg": 1e3 * float(np.mean([r["t_pcg"] for r in reps]))}


def _sweep_roofline(solver, hbm, peak_source):
    rf = solver.roofline()
    achieved = rf["bytes"] / rf["seconds"] / 1e9 if rf["seconds"] > 0 else 0.0
    return {"bound": "hbm", "kernel": rf["kernel"], "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "bytes_per_launch": rf["bytes"],
            "launch_ms": 1e3 * rf["seconds"], "peak_source": peak_source}


def _fp64_roofline(solver, peak):
    ft = solver.factor_timing()
    flops = ft["flops_cholesky"] + ft["flops_inverse"]
    achieved = flops / ft["seconds"] / 1e12 if ft["seconds"] > 0 else 0.0
    return {"bound": "tensor", "kernel": ft["kernel"], "achieved": achieved, "peak": peak["dmma_tflops"],
            "unit": "TFLOP/s", "frac": achieved / peak["dmma_tflops"], "traffic": None,
            "flops_per_launch": flops, "flops_cholesky": ft["flops_cholesky"], "flops_inverse_panels": ft["flops_inverse"],
            "launch_ms": 1e3 * ft["seconds"],
            "peak_source": "measured in this run: mma.sync.m8n8k4.f64 (DMMA.8x8x4) chains, peak.cu",
            "dfma_tflops": peak["dfma_tflops"]}


def _cfg5_leg(cb, args, hbm, peak_source, local):
    """BASELINE.json configs[4] on this GPU: one warm-up + 2 timed solves."""
    cfg = configs.get("cfg5")
    solver = cb.GpuSolver(local)
    pb = cb.prepare(solver, cfg)

    def step():
        solver.assemble(cfg.block, pb.block_ids)
        solver.setup_bddc(pb.objects, cfg.weighting)
        return solver.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)[1]
    step()
    tot, reps = _time_steps(step, 2)
    out = {"workload": f"cfg5-{cfg.cells}^3 (BASELINE.json configs[4], stiffness, cef)", "n_dof": pb.mesh.n_dof,
           "n_sd": len(pb.block_ids), "n_coarse": len(pb.objects), "iterations": reps[-1]["iterations"],
           "value": pb.mesh.n_dof * len(reps) / tot, "unit": "DOF/s", "steps": len(reps), "warmup": 1,
           "phases_ms": _phases(reps), "roofline": _sweep_roofline(solver, hbm, peak_source)}
    solver.close()
    return out


def _batch_leg(cfg, local, n_sys=8, conc=4):
    """a translation sweep of n_sys
    cfg4 systems, one at a time vs `conc` in flight (one handle and stream
    each); wall clock of the whole batch including each system's classify,
    partition, device objects, assembly, setup and PCG."""
    from paper_1703_06323_b200 import batch
    cfgs = batch.translation_sweep(cfg, n_sys)
    out = {"workload": f"{n_sys} translated {cfg.name} systems (eps in [-h, h] along (1,1,1)), warm handles"}
    for c in (1, conc):
        runner = batch.BatchRunner(local, c)
        runner.run(cfgs)  # warm: every handle's buffers and graphs exist
        res, wall = runner.run(cfgs)
        runner.close()
        nd = sum(r.n_dof for r in res)
        out[f"concurrency_{c}"] = {"value": nd / wall, "unit": "DOF/s", "wall_s": wall,
                                   "iterations": [r.report["iterations"] for r in res]}
    out["speedup"] = out[f"concurrency_{conc}"]["value"] / out["concurrency_1"]["value"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the cfg5 sub-measurement")
    ap.add_argument("--no-batch", action="store_true", help="skip the batched translation-sweep sub-measurement")
    args = ap.parse_args()
    rank, world, local = _env_rank()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch(args)
    if world != max(1, args.gpus):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
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
    else:
        solver = cb.GpuSolver(local)
        pb = cb.prepare(solver, cfg)
        lp = None
    mesh, block_ids, objs = pb.mesh, pb.block_ids, pb.objects
    n_dof = mesh.n_dof
    # the caller's BackgroundMesh arrays are page-locked once (cutbddc_host_pin):
    # the e2e uploads below are asynchronous DMA from pinned host memory
    pinned = [cb.pin(a) for a in (mesh.phi, mesh.cls, mesh.dof_of_node)]

    def assemble(s, mesh_view=None):  # the global partition; a distributed handle takes its own subdomains
        return s.assemble(cfg.block, block_ids, mesh=mesh_view)

    def step_device():
        assemble(solver)                                # mesh resident on the device
        solver.setup_bddc(objs, cfg.weighting)
        x, rep = solver.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
        return rep

    def solve_e2e(s):
        assemble(s, mesh)                                              # H2D of the mesh view
        o2 = s.classify_objects(cfg.objects, cfg.variant)              # objects (+ v1/v2 splits) on the device
        s.setup_bddc(o2, cfg.weighting)
        return s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)             # D2H of x

    def step_e2e():
        t0 = time.perf_counter()
        solve_e2e(solver)
        return time.perf_counter() - t0

    def step_e2e_fresh():  # one GPU only (a fresh NCCL communicator per solve is not measured)
        t0 = time.perf_counter()
        s = cb.GpuSolver(local)
        s.n_dof = n_dof
        solve_e2e(s)
        s.close()
        return time.perf_counter() - t0

    os.environ["CUTBDDC_NO_PLAN_CACHE"] = "1"          # cold task list in every timed step
    t_warm = time.perf_counter()
    for _ in range(args.warmup):
        rep = step_device()
    # beyond the W steps: keep solving (untimed) until the GPU has been busy for
    # about a second, so the timed region never starts on clocks still ramping
    # after an idle box (seen once: the first bench of a call 12% slower)
    extra_warm = 0
    while world == 1 and time.perf_counter() - t_warm < 1.0 and extra_warm < 200:
        step_device()
        extra_warm += 1
    if world > 1:
        dist.barrier()
    launches0 = solver.stats()["launches"]
    sampler = ClockSampler(local)
    sampler.start()
    tot, reps = _time_steps(step_device, args.steps)
    clocks = sampler.stop()
    launches = (solver.stats()["launches"] - launches0) / args.steps
    tot = _max_over_ranks(tot, world)
    value = n_dof * args.steps / tot                     # one global problem per step, solved by all ranks

    # numeric factorisation vs the FP64 tensor peak (last timed step's setup)
    peaks_fp64 = cb.fp64_peak(local)
    roof64 = _fp64_roofline(solver, peaks_fp64)

    # the same steps with the task-list cache on (repeated solves of one geometry)
    os.environ.pop("CUTBDDC_NO_PLAN_CACHE", None)
    step_device()
    wtot, wreps = _time_steps(step_device, args.steps)
    wtot = _max_over_ranks(wtot, world)
    os.environ["CUTBDDC_NO_PLAN_CACHE"] = "1"

    # e2e through the C ABI with host buffers: median of 5 wall-clock solves
    # (one host hiccup in a ~15 ms solve must not decide the number)
    step_e2e()
    e2e_t = sorted(step_e2e() for _ in range(5))
    e2e_med = _max_over_ranks(e2e_t[len(e2e_t) // 2], world)
    e2e = n_dof / e2e_med
    fresh = None
    if world == 1:
        step_e2e_fresh()
        ft = sorted(step_e2e_fresh() for _ in range(3))
        fresh = {"value": n_dof / ft[1], "unit": "DOF/s", "stat": "median of 3 solves, each on a new handle",
                 "samples_ms": [round(1e3 * t, 3) for t in ft]}
    n = cfg.cells
    obj_bytes = objs.dofs.nbytes + objs.neigh.nbytes + objs.kinds.nbytes + objs.dof_ptr.nbytes + objs.neigh_ptr.nbytes
    h2d = (n + 1) ** 3 * (8 + 4) + n ** 3 + 8 * len(block_ids) + obj_bytes  # mesh view, partition, coarse view
    d2h = 8 * n_dof + n_dof + obj_bytes  # solution, dirichlet mask, device-classified objects

    # roofline of the dominant PCG kernel family (triangular solves), timed live
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak_source = ("MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6.65 TB/s (B200_PROFILING.md)")
    roof = _sweep_roofline(solver, hbm, peak_source)
    # roofline.traffic: DRAM bytes of the same 7 sweep launches of one apply
    # from the committed ncu --set full capture (tools/ncu_traffic.py)
    for tname in ("r02_sweep_traffic_cfg4.json", "r01_sweep_traffic_cfg4.json"):
        tj = os.path.join(ROOT, "profiles", tname)
        if os.path.exists(tj) and world == 1 and cfg.name == "cfg4" and cfg.cells == 64:
            roof["traffic"] = json.load(open(tj))["traffic_bytes_per_apply"]
            roof["traffic_source"] = f"profiles/{tname} (ncu --set full, dram read+write)"
            break
    for a in pinned:
        cb.unpin(a)
    solver.close()

    cfg5 = None
    if world == 1 and not args.no_cfg5 and cfg.name == "cfg4":
        cfg5 = _cfg5_leg(cb, args, hbm, peak_source, local)

    batch_leg = None
    if world == 1 and not args.no_batch and cfg.name == "cfg4":
        batch_leg = _batch_leg(cfg, local)

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
            "phases_ms": _phases(reps),
            "step_ms": [round(1e3 * (r["t_assembly"] + r["t_setup"] + r["t_pcg"]), 3) for r in reps],
            "median_step_ms": float(np.median([r["t_assembly"] + r["t_setup"] + r["t_pcg"] for r in reps]) * 1e3),
            "extra_warmup_steps": extra_warm,
            "pcg_dofs_per_s": n_dof / np.mean([r["t_pcg"] for r in reps]),
            "timing": "every step rebuilds the factorisation task list (CUTBDDC_NO_PLAN_CACHE=1)",
            "warm": {"value": n_dof * args.steps / wtot, "unit": "DOF/s", "phases_ms": _phases(wreps),
                     "timing": "task-list cache on (repeated solves of one geometry)"},
            "roofline": roof, "roofline_fp64": roof64, "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "DOF/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "stat": "median of 5 solves", "samples_ms": [round(1e3 * t, 3) for t in e2e_t]},
            "e2e_fresh_handle": fresh, "cfg5": cfg5, "batch": batch_leg,
            "gpu_launches": int(launches), "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
