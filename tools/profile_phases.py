"""Per-phase device timing of one configuration (CUTBDDC_PROFILE=1 scopes):
warm solves, then a profiled assembly + setup + applies + solve sweeps."""
import os
import sys

os.environ["CUTBDDC_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
for _ in range(int(os.environ.get("PROFILE_REPS", "6"))):
    s.assemble(cfg.block, pb.block_ids)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
print({k: rep[k] for k in ("iterations", "t_assembly", "t_setup", "t_pcg")}, flush=True)
print(s.stats(), flush=True)
r = np.random.default_rng(0).uniform(-1, 1, s.n_dof)
for _ in range(3):
    s.apply(r)
print(s.roofline(reps=3), flush=True)
s.close()
