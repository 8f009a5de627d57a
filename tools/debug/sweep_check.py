"""Compare the dataflow sweeps with the level sweeps (local_solve hook)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

if len(sys.argv) > 2 and sys.argv[1] == "--child":
    from paper_1703_06323_b200 import configs, cutbddc as cb
    cfg = configs.get(sys.argv[2], weighting="stiffness", objects="cef")
    s = cb.GpuSolver(0)
    pb = cb.prepare(s, cfg)
    s.setup_bddc(pb.objects, cfg.weighting)
    sten, mi, mp, da, sd = s.local_system()
    rng = np.random.default_rng(3)
    out = {}
    for which, m in ((0, mi), (1, mp)):
        x = np.where(m > 0, rng.uniform(-1, 1, m.shape), 0.0)
        out[f"in{which}"] = x
        out[f"out{which}"] = s.local_solve(which, x)
    out["mi"], out["mp"] = mi, mp
    np.savez(sys.argv[3], **out)
    sys.exit(0)

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
res = {}
for mode in ("0", "1"):
    env = dict(os.environ, CUTBDDC_LEVEL_SWEEPS=mode)
    f = os.path.join(ROOT, "gpurun_out", f"sweep_{mode}.npz")
    subprocess.run([sys.executable, __file__, "--child", name, f], env=env, check=True)
    res[mode] = np.load(f)
for which in (0, 1):
    a, b = res["0"][f"out{which}"], res["1"][f"out{which}"]
    m = res["0"]["mi" if which == 0 else "mp"] > 0
    d = np.abs(a - b) * m
    rel = d.max() / max(1e-300, np.abs(b * m).max())
    print(f"which={which}: max rel diff {rel:.3e}; nan {np.isnan(a).sum()}")
    bad = np.argwhere(d > 1e-8 * np.abs(b * m).max())
    print("  bad (sd, slot) count", len(bad), "first", bad[:10].tolist())
    if len(bad):
        sds = np.unique(bad[:, 0])
        print("  subdomains with errors:", sds[:20].tolist(), "of", a.shape[0])
