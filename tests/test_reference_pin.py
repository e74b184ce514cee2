"""Pin the oracle and the product to the REFERENCE ITSELF.

tests/golden/ref_*.npz are outputs of the reference's own solver path
(/root/reference/proj/include/hosweep, compiled unmodified against the
Eigen-subset shim by `make -C oracle ref`; tests/golden/make_ref_golden.py).
They cover full C1, C1 with boundary inflow, and a reduced C2 (twisted 2D,
cyclic graphs): interior faces, per-ordinate couplings, edge weights, lag
flags, orders, cut sets, one lagged sweep per ordinate, local solves,
direct_oracle, converged source iteration and balance_report.

Encoding difference (not a result difference): FaceRecord::orientation is +1 /
-1 in the reference (mesh.hpp:47-53); the oracle and the product store a code,
0 (same direction) / 1 (reversed).
"""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_1810_11080_b200 as pk
from paper_1810_11080_b200 import problem as pb

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
CASES = {
    "ref_c1": ("c1", {}, {}),
    "ref_c1_inflow": ("c1", dict(cells=4), dict(inflow=0.7)),
    "ref_c2_small": ("c2", dict(cells=16, n_mu=2, n_az=8), {}),
    # FaceIntegration::Rule::romberg, the reference's default (assembly.hpp:33-40)
    "ref_c1_romberg": ("c1", {}, dict(face_rule=1)),
    "ref_c1_romberg_inflow": ("c1", dict(cells=4), dict(face_rule=1, inflow=0.7)),
    "ref_c2_small_romberg": ("c2", dict(cells=12, n_mu=2, n_az=8), dict(face_rule=1)),
}


def _case(name):
    cfg, kw, extra = CASES[name]
    prob = pb.config(cfg, **kw)
    if extra:
        prob = prob.replace(**extra)
    return prob, np.load(os.path.join(GOLD, name + ".npz"))


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _ref_faces(g):
    f = g["interior_faces"].reshape(-1, 5).copy()
    f[:, 4] = (f[:, 4] < 0).astype(f.dtype)   # +1 -> 0, -1 -> 1
    return f


def _check_plan(g, prob, couplings, ordering, faces):
    """Bit-exact: faces, couplings (face, downwind, upwind, lagged), edge weights,
    orders, cut sets and cut weights of every ordinate."""
    nd, ne = prob.num_ordinates, prob.num_elements
    assert np.array_equal(faces, _ref_faces(g))
    co = g["couplings"].reshape(-1, 4)
    off, lo = g["couplings_offsets"], g["lagged_offsets"]
    total = 0
    for d in range(nd):
        ints, w = couplings(d)
        assert np.array_equal(ints, co[off[d]:off[d + 1]]), d
        assert np.array_equal(w, g["edge_weights"][off[d]:off[d + 1]]), d   # FP64 bits
        order, lagged, lw = ordering(d)
        assert np.array_equal(order, g["order"][d * ne:(d + 1) * ne]), d
        assert np.array_equal(lagged, g["lagged_edges"][lo[d]:lo[d + 1]]), d
        assert lw == g["lagged_weight"][d], d
        total += len(lagged)
    assert total == int(g["total_lagged_edges"][0])
    return total


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_equals_reference(name):
    prob, g = _case(name)
    orc = O.OracleSolver(prob)
    nd, N = prob.num_ordinates, prob.num_dofs

    def ordering(d):
        o = orc.ordering(d)
        return o["order"], o["lagged_edges"], o["lagged_weight"]

    total = _check_plan(g, prob, orc.couplings, ordering, orc.interior_faces())
    assert total > 0   # cyclic graphs: the lagged path is exercised
    assert rel_l2(orc.sweep_all(g["phi"], g["psi_old"]), g["sweep"].reshape(nd, N)) <= 1e-13
    ls = np.stack([orc.local_solve(e, d, g["rhs"]) for d in range(nd) for e in (0, prob.num_elements - 1)])
    assert rel_l2(ls, g["local_solve"]) <= 1e-13
    ndir = g["direct_oracle"].size // N
    if ndir:
        do = np.stack([orc.direct_oracle(d, g["phi"]) for d in range(ndir)])
        assert rel_l2(do, g["direct_oracle"]) <= 1e-12
    its, conv = g["si_iterations"]
    r = orc.source_iteration(1e-12, 400, 0)
    assert r["converged"] and conv and r["iterations"] == its
    assert rel_l2(r["phi"], g["si_phi"]) <= 1e-12 and rel_l2(r["psi"], g["si_psi"].reshape(nd, N)) <= 1e-12
    np.testing.assert_allclose(r["error"], g["si_error"], rtol=1e-6, atol=1e-14)   # last entries: round-off level
    b = orc.balance(g["si_psi"].reshape(nd, N), g["si_phi"])
    for k, v in zip(("source_volume", "inflow", "absorption", "outflow"), g["balance"][:4]):
        assert abs(b[k] - v) <= 1e-12 * max(abs(v), 1.0), k
    assert b["outflow_by_attr"] == pytest.approx(dict(zip(g["balance_attrs"].tolist(),
                                                          g["balance_attr_outflow"].tolist())), rel=1e-12)


@pytest.mark.parametrize("name", sorted(CASES))
def test_product_plan_equals_reference(name):
    """The product's host plan (graph weights, Tarjan, FAS, Kahn; hsw_create with
    device < 0) equals the reference's, bit for bit."""
    prob, g = _case(name)
    s = pk.SweepSolver(prob, device=-1)

    def ordering(d):
        o = s.ordering(d)
        return o.order, o.lagged_edges, o.lagged_weight

    _check_plan(g, prob, s.couplings, ordering, s.interior_faces())
    assert s.total_lagged_edges() == int(g["total_lagged_edges"][0])


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include/hosweep"),
                    reason="the reference sources exist only in the build container")
def test_fixtures_regenerate_from_the_reference(tmp_path):
    """The committed fixtures are what the reference produces (rebuild + rerun)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("mrg", os.path.join(GOLD, "make_ref_golden.py"))
    mrg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mrg)
    subprocess.check_call(["make", "-s", "-C", os.path.join(os.path.dirname(HERE), "oracle"), "ref"])
    name, (cfg, kw), extra, tol, mx, ndir = mrg.CASES[0]
    prob = pb.config(cfg, **kw)
    out = mrg.run_case(prob, tol, mx, ndir)
    g = np.load(os.path.join(GOLD, name + ".npz"))
    for k in ("couplings", "edge_weights", "order", "lagged_edges", "sweep", "si_phi", "direct_oracle"):
        assert np.array_equal(out[k], g[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_equals_reference(name):
    """The B200 product against the reference's own outputs: plan bit-exact, one
    lagged sweep <= 1e-10, local solves, direct_oracle, converged SI <= 1e-8,
    balance_report."""
    prob, g = _case(name)
    nd, N = prob.num_ordinates, prob.num_dofs
    s = pk.SweepSolver(prob, pk.SolveOptions(tolerance=1e-12))

    def ordering(d):
        o = s.ordering(d)
        return o.order, o.lagged_edges, o.lagged_weight

    _check_plan(g, prob, s.couplings, ordering, s.interior_faces())
    assert rel_l2(s.sweep(-1, g["phi"], g["psi_old"]), g["sweep"].reshape(nd, N)) <= 1e-10
    for d in range(nd):
        assert rel_l2(s.sweep(d, g["phi"], g["psi_old"][d]), g["sweep"].reshape(nd, N)[d]) <= 1e-10
    ls = np.stack([s.local_solve(e, d, g["rhs"]) for d in range(nd) for e in (0, prob.num_elements - 1)])
    assert rel_l2(ls, g["local_solve"]) <= 1e-10
    ndir = g["direct_oracle"].size // N
    if ndir:
        do = np.stack([s.direct_oracle(d, g["phi"]) for d in range(ndir)])
        assert rel_l2(do, g["direct_oracle"]) <= 1e-10
    state, hist = s.source_iteration()
    its, conv = g["si_iterations"]
    assert hist.converged and hist.iterations() == its
    assert rel_l2(state.phi, g["si_phi"]) <= 1e-8 and rel_l2(state.psi, g["si_psi"].reshape(nd, N)) <= 1e-8
    per = g["si_per_ordinate"].reshape(its, nd)
    np.testing.assert_allclose(np.array(hist.per_ordinate), per, rtol=1e-5, atol=1e-14)
    b = pk.balance_report(s, state)
    for k, v in zip(("source_volume", "inflow", "absorption", "outflow"), g["balance"][:4]):
        assert abs(getattr(b, k) - v) <= 1e-10 * max(abs(v), 1.0), k
