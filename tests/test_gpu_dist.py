"""Distribution on the device (dist.cu): the exchange plan every rank builds
on its GPU equals the host plan (cutbddc_build_exchange_plan) entry for
entry — the plan the multi-process CPU tests (test_multigpu_gloo.py) drive
real exchanges with and prove bit-identical over 1-4 ranks. One GPU builds
every rank's view (a plan-only distribution: no communicator, no exchange)."""
import numpy as np
import pytest

from paper_1703_06323_b200 import configs
from paper_1703_06323_b200 import cutbddc as cb

pytestmark = pytest.mark.gpu


def _plans_equal(a, b):
    return (a.n_loc == b.n_loc and a.n_own == b.n_own and np.array_equal(a.loc_glob, b.loc_glob) and
            np.array_equal(a.seg_ptr, b.seg_ptr) and np.array_equal(a.copy_ptr, b.copy_ptr) and
            np.array_equal(a.copy_src, b.copy_src) and np.array_equal(a.nbr, b.nbr) and
            np.array_equal(a.send_ptr, b.send_ptr) and np.array_equal(a.send_src, b.send_src) and
            np.array_equal(a.recv_ptr, b.recv_ptr))


@pytest.mark.parametrize("name,world", [("cfg2", 1), ("cfg2", 2), ("cfg2", 4), ("cfg4", 2), ("cfg4", 8)])
def test_device_plan_equals_host_plan(name, world):
    cfg = configs.get(name)
    s = cb.GpuSolver(0)
    mesh = s.classify(cfg)
    block_ids = cb.build_partition(mesh, cfg.block)
    ros = cb.assign_subdomains(cfg.block, block_ids, cfg.cells, world)
    own = []
    for rank in range(world):
        s.set_distribution(cfg.block, block_ids, ros, rank, world)
        s.assemble(cfg.block, block_ids)
        dev = s.exchange_plan()
        host = cb.exchange_plan(mesh, cfg.block, block_ids, ros, rank, world)
        assert _plans_equal(dev, host), (name, world, rank)
        assert len(dev.seg_ptr) == int((ros == rank).sum()) + 1
        own.append(dev.loc_glob[:dev.n_own])
    assert np.array_equal(np.sort(np.concatenate(own)), np.arange(mesh.n_dof))
    s.close()


def test_plan_only_handle_refuses_numerics():
    cfg = configs.get("cfg2")
    s = cb.GpuSolver(0)
    mesh = s.classify(cfg)
    block_ids = cb.build_partition(mesh, cfg.block)
    ros = cb.assign_subdomains(cfg.block, block_ids, cfg.cells, 2)
    s.set_distribution(cfg.block, block_ids, ros, 1, 2)
    s.assemble(cfg.block, block_ids)
    with pytest.raises(cb.CutbddcError) as e:
        s.rhs()
    assert e.value.code == cb.CONFIG
    s.close()


def test_one_rank_plan_is_the_identity_layout():
    """One rank: every dof is local and owned, segments follow the lowest
    subdomain of each dof, and the sub-assembled SpMV equals the oracle's
    assembled Abar (matrix-free)."""
    from oracle.pyoracle import Oracle
    cfg = configs.get("cfg2", weighting="stiffness", objects="cef")
    s = cb.GpuSolver(0)
    pb = cb.prepare(s, cfg)
    p = s.exchange_plan()
    assert p.n_loc == p.n_own == pb.mesh.n_dof and len(p.nbr) == 0
    assert np.array_equal(np.sort(p.loc_glob), np.arange(pb.mesh.n_dof))
    o = Oracle(cfg)
    o.setup()
    x = np.random.default_rng(3).uniform(-1, 1, o.n_dof)
    y_o, y_g = o.spmv(x), s.spmv(x)
    assert np.linalg.norm(y_o - y_g) <= 1e-13 * np.linalg.norm(y_o)
    assert np.abs(o.rhs() - s.rhs()).max() <= 1e-13 * np.abs(o.rhs()).max()
    s.close()
