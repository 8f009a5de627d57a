"""Per-level timeline of CUTBDDC_SWEEP_TRACE dumps (template from a JSON list of [level, rows, cols])."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from trace_analyze import load  # noqa: E402

prefix, tplI, tplK = sys.argv[1], sys.argv[2], sys.argv[3]
for tag, tj in (("I_fwd", tplI), ("I_bwd", tplI), ("K_fwd", tplK), ("K_bwd", tplK)):
    sn = json.load(open(tj))
    items, tr = load(f"{prefix}_sweep{tag}.bin")
    t0 = tr[:, 0].min()
    lv = np.array([sn[s][0] for s in items[:, 1]])
    print(tag, f"span {(tr[:, 2].max() - t0) / 1e3:.1f} us")
    for L in sorted(set(lv)):
        m = lv == L
        k = np.bincount(items[m, 0], minlength=4)
        print(f"  L{L}: items {m.sum():5d} (S{k[0]} A{k[1]} C{k[2]} T{k[3]}) start {(tr[m, 0].min() - t0) / 1e3:6.1f} "
              f"deps-met med {np.median(tr[m, 1] - t0) / 1e3:6.1f} end {(tr[m, 2].max() - t0) / 1e3:6.1f} "
              f"work med {np.median(tr[m, 2] - tr[m, 1]) / 1e3:5.2f} max {(tr[m, 2] - tr[m, 1]).max() / 1e3:5.1f}")
