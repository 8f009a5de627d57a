"""Summarise CUTBDDC_DAG_TRACE dumps of the dataflow factorisation (dense_dag.cu):
per task kind wait / work times, and per template supernode (level of the
elimination tree) when its fronts' tasks ran."""
import glob
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from trace_analyze import load  # noqa: E402

NAMES = ["POTRF", "TRSM", "GEMM", "ACC", "FIN", "ASM", "PEN", "W", "DIAG"]


def load_fronts(path, n_tasks):
    with open(path, "rb") as f:
        f.seek(4 + 16 * n_tasks + 32 * n_tasks)
        raw = f.read(4)
        if len(raw) < 4:
            return None
        nf = int(np.frombuffer(raw, np.int32)[0])
        rec = np.frombuffer(f.read(80 * nf), np.int64).reshape(nf, 10)
    ints = rec[:, 3:].copy().view(np.int32).reshape(nf, 14)
    # r, c, np, nt, sd, sid, ch0, ch1, ntask, nasm, ntile, whole, grp, pad
    return ints


for p in sorted(glob.glob(sys.argv[1] + "_*.bin")):
    items, tr = load(p)
    kind = items[:, 0] >> 24
    fid = items[:, 0] & 0xFFFFFF
    t0 = tr[:, 0].min()
    print(f"{p}: {len(items)} tasks, {len(np.unique(fid))} fronts, span {(tr[:, 2].max() - t0) / 1e3:.1f} us, "
          f"SMs {len(np.unique(tr[:, 3]))}")
    for k, name in enumerate(NAMES):
        m = kind == k
        if not m.any():
            continue
        wait = (tr[m, 1] - tr[m, 0]) / 1e3
        work = (tr[m, 2] - tr[m, 1]) / 1e3
        print(f"  {name:5s} n={m.sum():6d} wait mean {wait.mean():7.2f} | work mean {work.mean():6.2f} p50 {np.median(work):6.2f} "
              f"max {work.max():7.2f} us | sum {work.sum() / 1e3:7.2f} ms")
    fr = load_fronts(p, len(items))
    if fr is None:
        continue
    key = fr[fid, 12] * 100000 + fr[fid, 5]
    print("  per supernode: grp  sid  fronts  whole  rows(max) cols(max)  first start  last end (us from launch)")
    for s in np.unique(key)[::-1]:
        m = key == s
        fm = fr[:, 12] * 100000 + fr[:, 5] == s
        print(f"    {s // 100000:3d} {s % 100000:4d} {fm.sum():6d} {fr[fm, 11].max():5d} {fr[fm, 0].max():8d} {fr[fm, 1].max():8d}"
              f"  {(tr[m, 0].min() - t0) / 1e3:10.1f} {(tr[m, 2].max() - t0) / 1e3:10.1f}")
