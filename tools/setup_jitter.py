"""Per-run device times of assembly / setup / PCG over repeated solves of one
configuration (run-to-run jitter of the dataflow launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
rows = []
for rep in range(int(os.environ.get("REPS", "12"))):
    s.assemble(cfg.block, pb.block_ids)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, r = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    rows.append((1e3 * r["t_assembly"], 1e3 * r["t_setup"], 1e3 * r["t_pcg"]))
for a, b, c in rows:
    print(f"assembly {a:6.2f}  setup {b:6.2f}  pcg {c:6.2f} ms")
s.close()
