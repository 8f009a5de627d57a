"""Summarise CUTBDDC_SWEEP_TRACE dumps of the dataflow sweeps (sweep.cu)."""
import glob
import sys

import numpy as np

KINDS = {0: "S", 1: "A", 2: "C", 3: "T"}


def load(path):
    with open(path, "rb") as f:
        n = int(np.frombuffer(f.read(4), np.int32)[0])
        items = np.frombuffer(f.read(16 * n), np.int32).reshape(n, 4)
        tr = np.frombuffer(f.read(32 * n), np.uint64).reshape(n, 4).astype(np.int64)
    return items, tr


def summarise(path):
    items, tr = load(path)
    t0 = tr[:, 0].min()
    span = (tr[:, 2].max() - t0) / 1e3
    print(f"{path}: {len(items)} items, span {span:.1f} us, SMs used {len(np.unique(tr[:, 3]))}")
    for k, name in KINDS.items():
        m = items[:, 0] == k
        if not m.any():
            continue
        wait = (tr[m, 1] - tr[m, 0]) / 1e3
        work = (tr[m, 2] - tr[m, 1]) / 1e3
        first = (tr[m, 0].min() - t0) / 1e3
        last = (tr[m, 2].max() - t0) / 1e3
        print(f"  {name}: n={m.sum():6d} wait mean {wait.mean():6.2f} max {wait.max():7.2f} | work mean {work.mean():6.2f} "
              f"p50 {np.median(work):6.2f} max {work.max():7.2f} us | active [{first:7.1f}, {last:7.1f}] us")
    # per supernode id: when its last item finished (critical path view)
    sids = np.unique(items[:, 1])
    rows = []
    for s in sids:
        m = items[:, 1] == s
        rows.append((int(s), int(m.sum()), (tr[m, 0].min() - t0) / 1e3, (tr[m, 2].max() - t0) / 1e3,
                     float(np.mean((tr[m, 2] - tr[m, 1]) / 1e3))))
    rows.sort(key=lambda r: r[3])
    print("  last 8 supernodes to finish (sid, items, first start, last end, mean work):")
    for r in rows[-8:]:
        print(f"    sn {r[0]:4d} items {r[1]:5d} start {r[2]:7.1f} end {r[3]:7.1f} work {r[4]:6.2f}")


if __name__ == "__main__":
    for p in sorted(glob.glob(sys.argv[1] + "*.bin")):
        summarise(p)
