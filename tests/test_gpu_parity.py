"""GPU parity: the CUDA sweep (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): per sweep relative L2 <= 1e-10; converged
source iteration <= 1e-8; integer graph/ordering work bit-exact.
"""
import math

import concurrent.futures

import numpy as np
import pytest

import oracle as O
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb

pytestmark = pytest.mark.gpu

SWEEP_TOL = 1e-10
SI_TOL = 1e-8


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _inputs(prob, seed=7):
    rng = np.random.default_rng(seed)
    N = prob.num_dofs
    phi = rng.uniform(0.0, 1.0, N)
    psi_old = rng.uniform(-0.5, 1.0, (prob.num_ordinates, N))
    return phi, psi_old


SMALL = [
    ("c1", {}),
    ("c2", dict(cells=16, n_mu=2, n_az=8)),
    ("c3", dict(cells=4, n_mu=2, n_az=4)),
    ("c4", dict(cells=4, n_mu=2, n_az=4)),
    ("c5", dict(cells=3, n_mu=2, n_az=4)),
]


@pytest.mark.parametrize("name,kw", SMALL, ids=[s[0] for s in SMALL])
def test_all_ordinate_sweep_matches_oracle(name, kw):
    prob = pb.config(name, **kw)
    gpu = pk.SweepSolver(prob)
    orc = O.OracleSolver(prob)
    phi, psi_old = _inputs(prob)
    got = gpu.sweep(-1, phi, psi_old)
    ref = orc.sweep_all(phi, psi_old)
    assert rel_l2(got, ref) <= SWEEP_TOL
    for d in range(prob.num_ordinates):
        assert rel_l2(got[d], ref[d]) <= SWEEP_TOL, d


@pytest.mark.parametrize("name,kw", SMALL[:3], ids=[s[0] for s in SMALL[:3]])
def test_single_ordinate_sweep_matches_oracle(name, kw):
    prob = pb.config(name, **kw)
    gpu = pk.SweepSolver(prob)
    orc = O.OracleSolver(prob)
    phi, psi_old = _inputs(prob, 11)
    for d in (0, prob.num_ordinates - 1):
        assert rel_l2(gpu.sweep(d, phi, psi_old[d]), orc.sweep(d, phi, psi_old[d])) <= SWEEP_TOL


def test_c1_one_sweep_from_zero_and_converged_si():
    """configs[0]: one sweep from psi=0, phi=0, then SI to ||dphi||/||phi|| < 1e-8."""
    prob = pb.config("c1")
    gpu = pk.SweepSolver(prob, pk.SolveOptions(tolerance=1e-8, criterion="phi_rel_l2"))
    orc = O.OracleSolver(prob)
    z = np.zeros(prob.num_dofs)
    zz = np.zeros((prob.num_ordinates, prob.num_dofs))
    assert rel_l2(gpu.sweep(-1, z, zz), orc.sweep_all(z, zz)) <= SWEEP_TOL
    state, hist = gpu.source_iteration()
    ref = orc.source_iteration(1e-8, 400, 1)
    assert hist.converged and ref["converged"]
    assert hist.iterations() == ref["iterations"]
    assert rel_l2(state.phi, ref["phi"]) <= SI_TOL
    assert rel_l2(state.psi, ref["psi"]) <= SI_TOL


def test_local_solve_and_hand_answer():
    # test_solver.cpp:40-54: 1 element, Omega=(1,0), sigma_t=1, q=1 -> cell average 4/11
    pts, nodes, bf = pb.generate_uniform(1, 1, 1)
    prob = pb.Problem(2, 1, 1, pts, nodes, np.ones(1, np.int32), bf, np.array([4 * math.pi]),
                      np.array([[1.0, 0.0, 0.5]]), {1: (1.0, 0.0)}, 0, (1.0,))
    s = pk.SweepSolver(prob)
    state, hist = s.source_iteration()
    assert hist.converged
    assert abs(state.psi[0].sum() / 4.0 - 4.0 / 11.0) < 1e-12
    # local solve residual vs the oracle's assembled block (test_solver.cpp:56-68)
    prob = pb.config("c2", cells=4, n_mu=2, n_az=4)
    s = pk.SweepSolver(prob)
    orc = O.OracleSolver(prob)
    rng = np.random.default_rng(17)
    for d in range(prob.num_ordinates):
        rhs = rng.uniform(-1, 1, prob.block_size)
        x = s.local_solve(3, d, rhs)
        A = orc.diag_block(3, d)
        assert np.abs(A @ x - rhs).max() < 1e-11 * np.abs(rhs).max()


def test_singular_block_reports_element_and_ordinate():
    # test_solver.cpp:332-344
    pts, nodes, bf = pb.generate_uniform(2, 1, 1, (0, 0, 2, 1))
    w, d = pb.level_symmetric_2d(2)
    prob = pb.Problem(2, 1, 1, pts, nodes, np.ones(2, np.int32), bf, w, d, {1: (1.0, 0.0)}, 0, (1.0,))
    s = pk.SweepSolver(prob)
    s.zero_block_for_test(0, 1)
    with pytest.raises(pk.SolverError, match=r"element 0.*ordinate 1"):
        s.sweep(-1, np.zeros(s.num_dofs), np.zeros((s.num_ordinates, s.num_dofs)))


def test_direct_oracle_matches_dense_global_solve():
    prob = pb.config("c1", cells=4)
    s = pk.SweepSolver(prob)
    orc = O.OracleSolver(prob)
    phi = np.full(prob.num_dofs, 0.3)
    for d in range(0, prob.num_ordinates, 3):
        assert rel_l2(s.direct_oracle(d, phi), orc.direct_oracle(d, phi)) < 1e-12


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_config_sweep_parity(name):
    prob = pb.config(name)
    gpu = pk.SweepSolver(prob)
    orc = O.OracleSolver(prob, cache_lu=False, check_rcond=False)
    phi, psi_old = _inputs(prob, 3)
    got = gpu.sweep(-1, phi, psi_old)
    ref = orc.sweep_all(phi, psi_old)
    assert rel_l2(got, ref) <= SWEEP_TOL


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_full_config_sampled_ordinates(name):
    prob = pb.config(name)
    gpu = pk.SweepSolver(prob)
    ds = [0, prob.num_ordinates // 2 + 3]
    orc = O.OracleSolver(prob, cache_lu=False, check_rcond=False, active=ds)
    phi, _ = _inputs(prob, 5)
    psi_olds = {d: np.random.default_rng(d).uniform(0, 1, prob.num_dofs) for d in ds}
    # the oracle's sweeps of distinct ordinates are independent (ctypes drops the GIL)
    with concurrent.futures.ThreadPoolExecutor(len(ds)) as pool:
        refs = dict(zip(ds, pool.map(lambda d: orc.sweep(d, phi, psi_olds[d]), ds)))
    for d in ds:
        assert rel_l2(gpu.sweep(d, phi, psi_olds[d]), refs[d]) <= SWEEP_TOL
        # graph / cut set / levels bit-exact
        oo = orc.ordering(d)
        so = gpu.ordering(d)
        assert (so.order == oo["order"]).all() and (so.lagged_edges == oo["lagged_edges"]).all()
        assert (so.level == oo["level"]).all()


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_singular_block_3d_production_kernels(name):
    """A zeroed local block is reported with its (element, ordinate) by each 3D
    production kernel (c3: one-warp DMMA, c4: DMMA with TMEM tiles, c5: register GJ)."""
    prob = pb.config(name, cells=2, n_mu=2, n_az=4)
    s = pk.SweepSolver(prob)
    s.zero_block_for_test(5, 3)
    with pytest.raises(pk.SolverError, match=r"element 5.*ordinate 3"):
        s.sweep(-1, np.zeros(s.num_dofs), np.zeros((s.num_ordinates, s.num_dofs)))


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_single_hex_element_all_orders(p):
    """Edge case: one twisted hexahedron (every face on the boundary), orders 1-4."""
    pts, nodes, bf = pb.generate_uniform_3d(1, 1, 1, p)
    pts = pb.twist_3d(pts, 0.7)
    w, d = pb.product_quadrature(3, 2, 4)
    prob = pb.Problem(3, p, p, pts, nodes, np.ones(1, np.int32), bf, w, d, {1: (2.0, 1.0)}, 0, (1.0,))
    gpu = pk.SweepSolver(prob)
    orc = O.OracleSolver(prob)
    phi, psi_old = _inputs(prob, 23)
    assert rel_l2(gpu.sweep(-1, phi, psi_old), orc.sweep_all(phi, psi_old)) <= SWEEP_TOL


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", dict(cells=24, n_mu=2, n_az=8)),
                                     ("c3", dict(cells=6, n_mu=4, n_az=8)), ("c4", dict(cells=6, n_mu=2, n_az=8)),
                                     ("c5", dict(cells=4, n_mu=2, n_az=8))])
def test_device_coupling_magnitudes_give_the_host_plan(name, kw):
    """the per-(ordinate, face) coupling magnitudes computed on
    the device drive edge existence and weights; the resulting graphs, cut sets,
    orders and levels equal the host-only plan bit for bit."""
    prob = pb.config(name, **kw)
    dev = pk.SweepSolver(prob)
    host = pk.SweepSolver(prob, device=-1)
    assert dev.total_lagged_edges() == host.total_lagged_edges()
    for d in range(prob.num_ordinates):
        a, b = dev.ordering(d), host.ordering(d)
        assert (a.order == b.order).all() and (a.position == b.position).all()
        assert (a.lagged_edges == b.lagged_edges).all() and a.lagged_weight == b.lagged_weight
        assert (a.level == b.level).all()
