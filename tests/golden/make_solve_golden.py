"""Golden oracle solves for the configs too large to re-run the CPU oracle
inside the GPU test session (tests/test_gpu_parity_b16.py): cfg4's
weak-scaling meshes 80^3 / 96^3 / 128^3 and cfg5 (256^3, {stiffness, cef}).

Each fixture holds the problem sizes, the PCG iteration count, the full
residual history, |x|, sum(x) and x at 2048 seeded sample indices, as
computed by the CPU restatement (oracle/). Run from the repo root:
    python tests/golden/make_solve_golden.py [cfg4_80 cfg4_96 cfg4_128 cfg5]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle  # noqa: E402
from paper_1703_06323_b200 import configs  # noqa: E402

CASES = {"cfg4_80": ("cfg4", 2), "cfg4_96": ("cfg4", 4), "cfg4_128": ("cfg4", 8), "cfg5": ("cfg5", 1)}


def make(key):
    name, gpus = CASES[key]
    cfg = configs.get(name, gpus=gpus)
    t0 = time.time()
    o = Oracle(cfg)
    o.setup()
    x, rep = o.pcg()
    info = o.info()
    idx = np.sort(np.random.default_rng(1703).choice(o.n_dof, size=min(2048, o.n_dof), replace=False))
    out = dict(config=f"{name} {cfg.cells}^3 objects={cfg.objects} weighting={cfg.weighting} variant={cfg.variant}",
               n_dof=o.n_dof, n_sd=info["n_sd"], n_coarse=info["n_coarse"], iterations=rep["iterations"],
               converged=bool(rep["converged"]), residuals=[float(v) for v in rep["residuals"]],
               x_norm=float(np.linalg.norm(x)), x_sum=float(x.sum()), sample_idx=idx.tolist(),
               sample_x=[float(v) for v in x[idx]], oracle_seconds=round(time.time() - t0, 1))
    fn = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"solve_{name}{'_' + str(cfg.cells) if name == 'cfg4' else ''}.json")
    json.dump(out, open(fn, "w"))
    print(key, out["n_dof"], out["iterations"], out["oracle_seconds"], "s ->", fn, flush=True)


if __name__ == "__main__":
    for k in sys.argv[1:] or list(CASES):
        make(k)
