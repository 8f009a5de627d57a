"""Per-run device times of assembly / setup / PCG over repeated solves of one
configuration (run-to-run jitter of the dataflow launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
if os.environ.get("SAMPLER"):  # A/B: the bench's clock sampler running alongside
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    smp = bench.ClockSampler(0)
    smp.start()
pb = cb.prepare(s, cfg)
rows = []
for rep in range(int(os.environ.get("REPS", "12"))):
    s.assemble(cfg.block, pb.block_ids)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, r = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    rows.append((1e3 * r["t_assembly"], 1e3 * r["t_setup"], 1e3 * r["t_pcg"]))
import numpy as np  # noqa: E402
r = np.array(rows)
print(f"reps {len(rows)} sampler={bool(os.environ.get('SAMPLER'))}: setup median {np.median(r[1:, 1]):.2f} mean "
      f"{r[1:, 1].mean():.2f} max {r[1:, 1].max():.2f} ms | pcg median {np.median(r[1:, 2]):.2f} ms")
s.close()
