"""Wall-clock breakdown of one end-to-end solve through the C ABI (the bench's
e2e step) next to the device-timed phases: where the host time goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
rows = []
for it in range(6):
    t = [time.perf_counter()]
    dirichlet = s.assemble(cfg.block, pb.block_ids, mesh=pb.mesh)
    t.append(time.perf_counter())
    if os.environ.get("HOST_OBJECTS"):
        o2 = cb.classify_objects(pb.mesh, cfg.block, pb.block_ids, dirichlet, cfg.objects, cfg.variant, None)
    else:
        o2 = s.classify_objects(cfg.objects, cfg.variant)
    t.append(time.perf_counter())
    s.setup_bddc(o2, cfg.weighting)
    t.append(time.perf_counter())
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    rows.append(list(d) + [1e3 * rep["t_assembly"], 1e3 * rep["t_setup"], 1e3 * rep["t_pcg"]])
r = np.median(np.array(rows[2:]), axis=0)
print(f"wall ms: assemble(H2D) {r[0]:.2f}  objects(host) {r[1]:.2f}  setup {r[2]:.2f}  pcg(+D2H) {r[3]:.2f}  "
      f"total {r[:4].sum():.2f}")
print(f"device ms: assembly {r[4]:.2f}  setup {r[5]:.2f}  pcg {r[6]:.2f}  total {r[4:].sum():.2f}")
s.close()
