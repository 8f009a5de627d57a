"""Median assembly / setup / PCG times of one configuration over a few solves
(for A/B runs of environment knobs: CUTBDDC_SPLIT_ROWS=... python tools/setup_sweep.py cfg4)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
ta, ts, tp = [], [], []
for _ in range(reps):
    s.assemble(cfg.block, pb.block_ids)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, r = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    ta.append(r["t_assembly"]), ts.append(r["t_setup"]), tp.append(r["t_pcg"])
m = lambda v: 1e3 * float(np.median(v[1:]))  # noqa: E731
tot = m(ta) + m(ts) + m(tp)
print(f"{cfg.name} iters {r['iterations']} assembly {m(ta):.2f} setup {m(ts):.2f} pcg {m(tp):.2f} ms "
      f"-> {pb.mesh.n_dof / tot / 1e3:.2f} M DOF/s", flush=True)
s.close()
