"""Product host layer (libcutbddc.so, no GPU needed): partition and interface
objects must equal the oracle's index maps bit for bit;
the library must export every symbol include/cutbddc.h declares."""
import os
import re

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_1703_06323_b200 import configs
from paper_1703_06323_b200 import cutbddc as cb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_match_header():
    hdr = open(os.path.join(ROOT, "include", "cutbddc.h")).read()
    declared = set(re.findall(r"\b(cutbddc_[a-z0-9_]+)\s*\(", hdr))
    lib = cb.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(cb.EXPORTS)


def _mesh_from_oracle(o):
    phi, cls, dof = o.mesh()
    c = o.cfg
    return cb.Mesh(c.cells, tuple(c.lo), (c.hi[0] - c.lo[0]) / c.cells, phi, cls, dof, o.n_dof)


@pytest.mark.parametrize("name,kw", [("cfg1", {}), ("cfg2", dict(objects="cef")), ("cfg3", {}),
                                     ("cfg2", dict(objects="cef", variant="v1", weighting="stiffness")),
                                     ("cfg2", dict(objects="cef", variant="v2", weighting="stiffness"))])
def test_objects_bit_exact_vs_oracle(name, kw):
    cfg = configs.get(name, **kw)
    o = Oracle(cfg)
    o.setup()
    mesh = _mesh_from_oracle(o)
    ids = cb.build_partition(mesh, cfg.block)
    exp_ids = [o.subdomain(s)["block_id"] for s in range(o.info()["n_sd"])]
    assert ids.tolist() == exp_ids
    diag = None
    if cfg.variant == configs.V2:
        parts = []
        for s in range(len(ids)):
            d = o.subdomain(s)
            import scipy.sparse as sp
            n = len(d["l2g"])
            parts.append(sp.csr_matrix((d["val"], d["col"], d["ptr"]), shape=(n, n)).diagonal())
        diag = np.ascontiguousarray(np.concatenate(parts))
    objs = cb.classify_objects(mesh, cfg.block, ids, o.dirichlet(), cfg.objects, cfg.variant, diag)
    assert objs.as_list() == o.objects(1)


def test_partition_rejects_indivisible():
    o = Oracle(configs.get("cfg1"), block=0)
    with pytest.raises(cb.CutbddcError) as e:
        cb.build_partition(_mesh_from_oracle(o), 7)
    assert e.value.code == cb.INVALID_ARGUMENT
