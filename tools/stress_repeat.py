"""Race hunt for the dataflow kernels: many repeated solves (and applies on a
random vector) of one configuration must return identical bits every time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = configs.get(name)
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
s.setup_bddc(pb.objects, cfg.weighting)
r = np.random.default_rng(1).uniform(-1, 1, s.n_dof)
z0 = s.apply(r)
x0, rep0 = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
bad = 0
for k in range(reps):
    if k % 3 == 0:  # a fresh factorisation now and then
        s.assemble(cfg.block, pb.block_ids)
        s.setup_bddc(pb.objects, cfg.weighting)
    z = s.apply(r)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    if not (np.array_equal(z, z0) and np.array_equal(x, x0) and rep["iterations"] == rep0["iterations"]):
        bad += 1
        print("MISMATCH at repetition", k, np.abs(z - z0).max(), np.abs(x - x0).max(), rep["iterations"], flush=True)
print(f"{name}: {reps} repetitions, {bad} mismatches, iterations {rep0['iterations']}")
s.close()
sys.exit(1 if bad else 0)
