"""Solve one configuration on the GPU and print sizes, timings and convergence."""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
kw = dict(a.split("=") for a in sys.argv[2:])
cfg = configs.get(name, **kw)
t0 = time.perf_counter()
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
t1 = time.perf_counter()
print(f"{name} {kw}: n_dof {pb.mesh.n_dof}, subdomains {len(pb.block_ids)}, coarse objects {len(pb.objects)}; "
      f"host prepare {t1 - t0:.2f} s", flush=True)
for rep in range(2):
    s.assemble(cfg.block, pb.block_ids)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, r = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    print(f"  run {rep}: iterations {r['iterations']} converged {r['converged']} cond {r['cond']:.3g} | assembly "
          f"{1e3 * r['t_assembly']:.1f} ms setup {1e3 * r['t_setup']:.1f} ms pcg {1e3 * r['t_pcg']:.1f} ms | "
          f"{pb.mesh.n_dof / (r['t_assembly'] + r['t_setup'] + r['t_pcg']) / 1e6:.2f} M DOF/s", flush=True)
print(s.stats())
