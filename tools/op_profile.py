"""One configuration set up, then the iteration pieces timed once each
(an ncu target for the matrix-free operator: -k regex:k_sub_apply)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
s.setup_bddc(pb.objects, cfg.weighting)
print(s.time_parts(reps=1))
s.close()
