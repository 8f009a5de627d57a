"""Host hiccups in the timed steps: N cold-plan solves of cfg4 without the
bench's clock sampler, with it at 20 ms, and at 100 ms; per leg the median
step, the mean, and the steps slower than 1.2x the median."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

os.environ["CUTBDDC_NO_PLAN_CACHE"] = "1"
cfg = configs.get("cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
N = int(os.environ.get("REPS", "300"))


def leg(name, period, nogc=False):
    smp = None
    if period:
        smp = bench.ClockSampler(0)
        smp.period = period
        smp.start()
    if nogc:
        gc.disable()
    rows, wall = [], []
    for _ in range(N):
        t0 = time.perf_counter()
        s.assemble(cfg.block, pb.block_ids)
        s.setup_bddc(pb.objects, cfg.weighting)
        x, r = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
        wall.append(1e3 * (time.perf_counter() - t0))
        rows.append(1e3 * (r["t_assembly"] + r["t_setup"] + r["t_pcg"]))
    if nogc:
        gc.enable()
    n_s = len(smp.rows) if smp else 0
    if smp:
        smp.stop()
    r = np.array(rows)
    med = np.median(r)
    slow = r[r > 1.2 * med]
    print(f"{name:28s} median {med:.3f} mean {r.mean():.3f} ms | {len(slow)} slow steps {np.round(np.sort(slow)[-6:], 1).tolist()} "
          f"| wall median {np.median(wall):.3f} | samples {n_s}", flush=True)


for _ in range(20):
    s.assemble(cfg.block, pb.block_ids)
    s.setup_bddc(pb.objects, cfg.weighting)
    s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
leg("no sampler", 0)
leg("sampler 20 ms", 0.02)
leg("sampler 100 ms", 0.1)
leg("no sampler, gc off", 0, nogc=True)
leg("sampler 100 ms, gc off", 0.1, nogc=True)
leg("no sampler (again)", 0)
s.close()
