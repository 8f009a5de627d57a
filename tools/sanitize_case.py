"""One small solve through the C ABI (classify, assemble, device objects,
BDDC setup, PCG) for compute-sanitizer runs: tools/gpu_safety.sh."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
kw = dict(a.split("=") for a in sys.argv[2:])
cfg = configs.get(name, **kw)
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
objs = s.classify_objects(cfg.objects, 0) if cfg.variant == configs.V_STANDARD else pb.objects
s.setup_bddc(objs, cfg.weighting)
x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
assert rep["converged"], rep
print(f"{name} {kw}: n_dof {pb.mesh.n_dof} iterations {rep['iterations']}", flush=True)
s.close()
