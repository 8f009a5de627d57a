"""Summarise CUTBDDC_DAG_TRACE dumps of the dense-front DAG (dense_dag.cu)."""
import glob
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from trace_analyze import load  # noqa: E402

NAMES = ["POTRF", "TRSM", "GEMM", "ACC", "FIN"]
for p in sorted(glob.glob(sys.argv[1] + "_*.bin")):
    items, tr = load(p)
    kind = items[:, 0] >> 24
    t0 = tr[:, 0].min()
    print(f"{p}: {len(items)} tasks, {len(np.unique(items[:, 0] & 0xffffff))} fronts, span {(tr[:, 2].max() - t0) / 1e3:.1f} us")
    for k, name in enumerate(NAMES):
        m = kind == k
        if not m.any():
            continue
        wait = (tr[m, 1] - tr[m, 0]) / 1e3
        work = (tr[m, 2] - tr[m, 1]) / 1e3
        print(f"  {name:5s} n={m.sum():6d} wait mean {wait.mean():7.2f} | work mean {work.mean():6.2f} p50 {np.median(work):6.2f} "
              f"max {work.max():7.2f} us | sum {work.sum() / 1e3:7.2f} ms")
