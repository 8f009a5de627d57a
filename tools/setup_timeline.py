"""Timeline of one warm assembly + setup + PCG (CUTBDDC_PROFILE=2): every
profiled scope in order with its device start/duration and host start/duration
(ms from the first scope), to see where the device waits on host work."""
import os
import sys

os.environ["CUTBDDC_PROFILE"] = "2"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
for _ in range(3):
    s.assemble(cfg.block, pb.block_ids)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
print({k: rep[k] for k in ("iterations", "t_assembly", "t_setup", "t_pcg")}, flush=True)
s.close()
