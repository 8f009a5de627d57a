"""Warm per-piece device timing of one PCG iteration (cutbddc_gpu_time_parts)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

for name in (sys.argv[1:] or ["cfg4"]):
    cfg = configs.get(name)
    s = cb.GpuSolver(0)
    pb = cb.prepare(s, cfg)
    s.setup_bddc(pb.objects, cfg.weighting)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    x, rep = s.pcg(rtol=cfg.rtol, max_iter=cfg.max_iter)
    print(name, "iterations", rep["iterations"], "pcg ms", round(1e3 * rep["t_pcg"], 3),
          "per iteration us", round(1e6 * rep["t_pcg"] / rep["iterations"], 1), flush=True)
    print({k: round(v, 1) for k, v in s.time_parts().items()}, flush=True)
    s.close()
