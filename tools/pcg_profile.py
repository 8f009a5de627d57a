"""One cfg4 solve for an ncu launch list of the PCG loop (run with
CUTBDDC_NO_WHILE_GRAPH=1 so every iteration is a plain graph launch whose
kernel nodes ncu lists one by one): tools/gpu_pcg_profile.sh."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
s.setup_bddc(pb.objects, cfg.weighting)
x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
print("iterations", rep["iterations"], flush=True)
s.close()
