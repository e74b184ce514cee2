"""FaceIntegration::Rule::romberg — the reference's DEFAULT face rule
(assembly.hpp:33-40, :121-131; romberg.hpp:33-88), 2D as the reference.

The reference-generated pins (oracle and product plan bit-exact, GPU sweep / SI /
balance) are in test_reference_pin.py (ref_*_romberg fixtures).  Here: the
reference's own known-answer test "Romberg and Gauss face assembly agree on
straight meshes" (test_assembly.cpp:161-175), for the oracle's blocks and for the
product (host plan weights on CPU; sweeps on the GPU)."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb


def _straight(face_rule, face_points=0, omega=(0.8688903, 0.3500212)):
    pts, nodes, bf = pb.generate_uniform(3, 2, 2, rect=(0.0, 0.0, 1.5, 1.0))
    n = math.hypot(*omega)
    d = np.array([[omega[0], omega[1], math.sqrt(max(0.0, 1.0 - n * n))]])
    return pb.Problem(2, 2, 2, pts, nodes, np.ones(len(nodes), np.int32), bf, np.array([4 * math.pi]), d,
                      {1: (1.0, 0.5)}, 0, (1.0,), face_rule=face_rule, face_points=face_points, inflow=0.3)


def test_oracle_romberg_equals_gauss_on_straight_mesh():
    a = O.OracleSolver(_straight(1))
    b = O.OracleSolver(_straight(0, face_points=8))
    ia, wa = a.couplings(0)
    ib, wb = b.couplings(0)
    assert np.array_equal(ia, ib)
    for c in range(len(ia)):
        assert np.abs(a.coupling_block(0, c) - b.coupling_block(0, c)).max() < 1e-12
    for e in range(a.nel):
        assert np.abs(a.diag_block(e, 0) - b.diag_block(e, 0)).max() < 1e-12   # outflow enters the diagonal
    assert np.abs(a.source(0)[1] - b.source(0)[1]).max() < 1e-12             # boundary inflow moments


def test_product_plan_romberg_equals_gauss_on_straight_mesh():
    a = pk.SweepSolver(_straight(1), device=-1)
    b = pk.SweepSolver(_straight(0, face_points=8), device=-1)
    ia, wa = a.couplings(0)
    ib, wb = b.couplings(0)
    assert np.array_equal(ia, ib)
    np.testing.assert_allclose(wa, wb, rtol=0, atol=1e-12)


def test_romberg_is_2d_only():
    prob = pb.config("c3", cells=2, n_mu=2, n_az=4).replace(face_rule=1)
    with pytest.raises(ValueError, match="2D"):   # invalid argument (the reference has no 3D)
        pk.SweepSolver(prob, device=-1)


@pytest.mark.gpu
def test_gpu_romberg_equals_gauss_on_straight_mesh():
    a = pk.SweepSolver(_straight(1))
    b = pk.SweepSolver(_straight(0, face_points=8))
    rng = np.random.default_rng(5)
    phi = rng.uniform(0, 1, a.num_dofs)
    psi_old = rng.uniform(0, 1, (1, a.num_dofs))
    x, y = a.sweep(-1, phi, psi_old), b.sweep(-1, phi, psi_old)
    assert np.abs(x - y).max() <= 1e-12 * np.abs(y).max()


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", dict(cells=20, n_mu=2, n_az=8))])
def test_gpu_romberg_sweep_and_si_match_oracle(name, kw):
    """Twisted meshes (curved faces, partially outflow faces): the GPU with the Romberg
    blocks against the oracle's Romberg restatement, one sweep <= 1e-10 and converged SI."""
    prob = pb.config(name, **kw).replace(face_rule=1, inflow=0.4)
    s = pk.SweepSolver(prob, pk.SolveOptions(tolerance=1e-12))
    orc = O.OracleSolver(prob)
    nd, N = prob.num_ordinates, prob.num_dofs
    rng = np.random.default_rng(8)
    phi = rng.uniform(0, 1, N)
    psi_old = rng.uniform(-0.5, 1, (nd, N))
    got = s.sweep(-1, phi, psi_old)
    ref = orc.sweep_all(phi, psi_old)
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    state, hist = s.source_iteration()
    r = orc.source_iteration(1e-12, 400, 0)
    assert hist.converged and hist.iterations() == r["iterations"]
    assert np.linalg.norm(state.phi - r["phi"]) <= 1e-8 * np.linalg.norm(r["phi"])


@pytest.mark.gpu
@pytest.mark.parametrize("face_points", [2, 8])
def test_gpu_gauss_other_point_counts_match_oracle(face_points):
    """FaceIntegration::gauss_points other than the kernels' own p + 2 (the reference's
    default is 8): the faces are integrated at create and the kernels take the blocks."""
    prob = pb.config("c2", cells=10, n_mu=2, n_az=8).replace(face_points=face_points, inflow=0.2)
    s = pk.SweepSolver(prob)
    orc = O.OracleSolver(prob)
    for d in range(prob.num_ordinates):
        o = s.ordering(d)
        r = orc.ordering(d)
        assert (o.order == r["order"]).all() and (o.lagged_edges == r["lagged_edges"]).all()
    rng = np.random.default_rng(2)
    phi = rng.uniform(0, 1, prob.num_dofs)
    psi_old = rng.uniform(0, 1, (prob.num_ordinates, prob.num_dofs))
    got, ref = s.sweep(-1, phi, psi_old), orc.sweep_all(phi, psi_old)
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw,extra", [("c1", {}, dict(face_rule=1, inflow=0.3)),
                                           ("c3", dict(cells=4, n_mu=2, n_az=4), dict(inflow=0.3)),
                                           ("c2", dict(cells=12, n_mu=2, n_az=8), {})])
def test_device_balance_report_matches_oracle(name, kw, extra):
    """balance_report (solver.hpp:220-245) evaluated on the device from the resident
    converged state (hsw_balance_resident) against the oracle's and the host path's."""
    prob = pb.config(name, **kw).replace(**extra)
    s = pk.SweepSolver(prob, pk.SolveOptions(tolerance=1e-12, max_iterations=3000))
    state, hist = s.source_iteration()
    assert hist.converged
    dev = pk.balance_report(s)                        # resident: device path
    host = pk.balance_report(s, pk.SolverState(state.psi.copy(), state.phi.copy(), state.iterations))
    bo = O.OracleSolver(prob).balance(state.psi, state.phi)
    for k in ("source_volume", "inflow", "absorption", "outflow"):
        assert abs(getattr(dev, k) - bo[k]) <= 1e-10 * max(abs(bo[k]), 1e-300), k
        assert abs(getattr(dev, k) - getattr(host, k)) <= 1e-12 * max(abs(bo[k]), 1e-300), k
    assert abs(dev.residual) <= 1e-8 * bo["source_total"]
    for a, v in bo["outflow_by_attr"].items():
        assert abs(dev.outflow_by_attr[a] - v) <= 1e-10 * abs(bo["outflow"])
