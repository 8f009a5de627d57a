"""One cfg4 setup + a few BDDC applies (for ncu launch lists of the apply)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
s.setup_bddc(pb.objects, cfg.weighting)
r = np.random.default_rng(0).uniform(-1, 1, s.n_dof)
for _ in range(3):
    s.apply(r)
print(s.roofline(reps=5))
