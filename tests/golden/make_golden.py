"""Generate tests/golden/classification.json from the REFERENCE's own
classification code (levelset.cpp + mesh.cpp compiled unmodified into
oracle/_ref/libref.so by oracle/ref.mk). Run here (needs /root/reference):

    make -C oracle -f ref.mk && python tests/golden/make_golden.py

The fixture stores, per case, the counts and SHA-256 digests of the snapped
node phi (float64), the cell classes (uint8) and dof_of_node (int32) arrays,
so the GPU box can check bit-exactness without /root/reference.
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1703_06323_b200 import configs  # noqa: E402

CASES = ["sphere-id1", "sphere-id2", "sphere-id3", "sphere-id4", "cfg1", "cfg2"]


def case_cfg(name):
    if name.startswith("sphere-id"):
        return configs.sphere_id(int(name[-1]))
    return configs.get(name)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref.so"))
    out = {}
    for name in CASES:
        cfg = case_cfg(name)
        assert len(cfg.balls) == 1
        cx, cy, cz, r = cfg.balls[0]
        n = cfg.cells
        nn, nc = (n + 1) ** 3, n ** 3
        phi = np.zeros(nn)
        cls = np.zeros(nc, np.uint8)
        dof = np.zeros(nn, np.int32)
        ndof = C.c_longlong()
        cells = (C.c_int * 3)(n, n, n)
        lo = (C.c_double * 3)(*cfg.lo)
        hi = (C.c_double * 3)(*cfg.hi)
        cen = (C.c_double * 3)(cx, cy, cz)
        rc = lib.ref_classify(cells, lo, hi, cen, C.c_double(r), phi.ctypes.data_as(C.POINTER(C.c_double)),
                              cls.ctypes.data_as(C.POINTER(C.c_ubyte)), dof.ctypes.data_as(C.POINTER(C.c_int)),
                              C.byref(ndof))
        assert rc == 0
        out[name] = dict(cells=n, n_dof=int(ndof.value), n_interior=int((cls == 0).sum()),
                         n_exterior=int((cls == 1).sum()), n_cut=int((cls == 2).sum()),
                         sha_phi=sha(phi), sha_cls=sha(cls), sha_dof_of_node=sha(dof))
        print(name, out[name]["n_dof"], out[name]["n_cut"])
    with open(os.path.join(ROOT, "tests", "golden", "classification.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
